// Generic element-wise expression evaluation: the reference's eval_pointwise
// (state.hpp:126-193) over eval_expr (expr.hpp:186-222), for any ExprDag the
// DSL can express. The three fused patterns of the paper have dedicated
// kernels (fused_opt.cu, fused_bdr.cu); this interpreter is what GpuEngine
// uses for every other Pointwise / fused expression, so any ccopt program runs
// on the device with the reference's exact semantics:
//   * IEEE double, no contraction (explicit _rn intrinsics), nodes evaluated
//     once per element in DAG order (the memo of eval_expr);
//   * Update stores float(v) into its target at the element and yields the
//     unrounded v (expr.hpp:207-211);
//   * ReduceTensor values come from a pre-pass (coconet_pointwise_reduce);
//   * operands are read through BroadcastView (view.hpp:75-98) and, when
//     sliced, DistView::to_local (view.hpp:49-60).
#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.h"

using namespace coconet;

namespace {

constexpr int kThreads = 256;
constexpr int kReduceBlocks = 512;

struct LocalRanks {
  char* base[kMaxRanks];  // heap of each local rank
  int rank[kMaxRanks];    // its group-relative rank
  int world;              // group size
};

__device__ __forceinline__ double load_elem(const char* p, int elem, int64_t i) {
  switch (elem) {
    case COCONET_F16: return double(__half2float(reinterpret_cast<const __half*>(p)[i]));
    case COCONET_BF16: return double(__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]));
    default: return double(reinterpret_cast<const float*>(p)[i]);
  }
}

__device__ __forceinline__ void store_elem(char* p, int elem, int64_t i, double v) {
  const float f = float(v);
  switch (elem) {
    case COCONET_F16: reinterpret_cast<__half*>(p)[i] = __float2half_rn(f); break;
    case COCONET_BF16: reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(f); break;
    default: reinterpret_cast<float*>(p)[i] = f;
  }
}

__device__ __forceinline__ int64_t numel(const coconet_operand& o) {
  int64_t n = 1;
  for (int d = 0; d < o.ndim; ++d) n *= o.shape[d];
  return n;
}

// DistView::to_local for an operand sliced on o.sliced_dim
__device__ __forceinline__ int64_t to_local(const coconet_operand& o, int64_t g, int W) {
  if (o.sliced_dim < 0) return g;
  const int d = o.sliced_dim;
  int64_t st = 1;
  for (int i = d + 1; i < o.ndim; ++i) st *= o.shape[i];
  const int64_t ext = o.shape[d], per = ext / W;
  const int64_t before = g / (st * ext);
  const int64_t c = (g / st) % ext;
  const int64_t after = g % st;
  return (before * per + c % per) * st + after;
}

// DistView::to_global for the iteration space (the output)
__device__ __forceinline__ int64_t to_global(const coconet_expr_program& p, int rank, int64_t li, int W) {
  if (p.out_sliced_dim < 0) return li;
  const int d = p.out_sliced_dim;
  int64_t st = 1;
  for (int i = d + 1; i < p.out_ndim; ++i) st *= p.out_shape[i];
  const int64_t ext = p.out_shape[d], per = ext / W;
  const int64_t before = li / (st * per);
  const int64_t lc = (li / st) % per;
  const int64_t after = li % st;
  return (before * ext + int64_t(rank) * per + lc) * st + after;
}

// BroadcastView::map: output flat index -> operand flat index (trailing axes
// aligned, extent-1 axes stretched)
__device__ __forceinline__ int64_t bmap(const coconet_expr_program& p, const coconet_operand& o, int64_t g) {
  int64_t in = 0, in_stride = 1, rem = g;
  const int off = p.out_ndim - o.ndim;
  for (int d = p.out_ndim - 1; d >= 0; --d) {
    const int64_t ext = p.out_shape[d];
    const int64_t c = rem % ext;
    rem /= ext;
    if (d >= off) {
      const int64_t ie = o.shape[d - off];
      if (!(ie == 1 && ext != 1)) in += c * in_stride;
      in_stride *= ie;
    }
  }
  return in;
}

__device__ __forceinline__ double read_operand(const coconet_expr_program& p, const coconet_operand& o,
                                               const char* base, int64_t g, int W) {
  const int64_t ig = bmap(p, o, g);
  return load_elem(base + o.off, o.elem, to_local(o, ig, W));
}

// Evaluates the node list at one element; returns the root value. `write`
// enables Update stores (the per-element pass) — the ReduceTensor pre-pass
// evaluates with ctx.write unset (state.hpp:145-150).
__device__ double eval_element(const coconet_expr_program& p, char* base, int rank, int64_t g, int W,
                               const double* consts, const double* reduced, bool write) {
  double v[COCONET_EXPR_MAX_NODES];
  for (int i = 0; i < p.n_nodes; ++i) {
    const coconet_expr_node& n = p.nodes[i];
    double x = 0.0;
    switch (n.op) {
      case COCONET_OP_CONST: x = n.slot >= 0 ? consts[n.slot] : n.value; break;
      case COCONET_OP_INPUT: x = read_operand(p, p.inputs[n.slot], base, g, W); break;
      case COCONET_OP_ADD: x = __dadd_rn(v[n.a], v[n.b]); break;
      case COCONET_OP_SUB: x = __dsub_rn(v[n.a], v[n.b]); break;
      case COCONET_OP_MUL: x = __dmul_rn(v[n.a], v[n.b]); break;
      case COCONET_OP_DIV: x = __ddiv_rn(v[n.a], v[n.b]); break;
      case COCONET_OP_SQRT: x = __dsqrt_rn(v[n.a]); break;
      case COCONET_OP_POW: x = pow(v[n.a], v[n.b]); break;  // element-varying pow only
      case COCONET_OP_DROPOUT: {
        const bool keep = counter_uniform(p.seed, n.key, uint64_t(g)) >= n.rate;
        x = keep ? __ddiv_rn(v[n.a], 1.0 - n.rate) : 0.0;
        break;
      }
      case COCONET_OP_REDUCED: x = reduced[n.slot]; break;
      case COCONET_OP_UPDATE: {
        x = v[n.a];
        if (write) {
          const coconet_operand& t = p.targets[n.slot];
          store_elem(base + t.off, t.elem, to_local(t, g, W), x);
        }
        break;
      }
    }
    v[i] = x;
  }
  return v[p.root];
}

__global__ void __launch_bounds__(kThreads) pointwise_kernel(const coconet_expr_program p, LocalRanks lr,
                                                             const double* consts, const double* reduced) {
  const int li_rank = blockIdx.y;
  const int rank = lr.rank[li_rank];
  char* base = lr.base[li_rank];
  const int W = lr.world;
  const int64_t n_local = p.out_sliced_dim >= 0 ? numel(p.out) / W : numel(p.out);
  const double* cr = consts + int64_t(li_rank) * p.n_rank_consts;
  const double* rr = reduced + int64_t(li_rank) * p.n_reduce;
  for (int64_t li = int64_t(blockIdx.x) * kThreads + threadIdx.x; li < n_local; li += int64_t(gridDim.x) * kThreads) {
    const int64_t g = to_global(p, rank, li, W);
    const double y = eval_element(p, base, rank, g, W, cr, rr, true);
    store_elem(base + p.out.off, p.out.elem, li, y);
  }
}

// reduce pass: per-block partials in a fixed order, then one block per rank
// folds them in block order (deterministic).
__device__ __forceinline__ double fold(int red, double a, double b) {
  return red == COCONET_SUM ? a + b : (red == COCONET_MAX ? (a > b ? a : b) : (a < b ? a : b));
}

__global__ void __launch_bounds__(kThreads) pointwise_reduce_kernel(const coconet_expr_program p, LocalRanks lr,
                                                                    const double* consts, int red,
                                                                    double* block_part, int* block_has) {
  __shared__ double s_v[kThreads];
  __shared__ int s_h[kThreads];
  const int li_rank = blockIdx.y;
  const int rank = lr.rank[li_rank];
  char* base = lr.base[li_rank];
  const int W = lr.world;
  const int64_t n_local = p.out_sliced_dim >= 0 ? numel(p.out) / W : numel(p.out);
  const double* cr = consts + int64_t(li_rank) * p.n_rank_consts;
  double acc = 0.0;
  int has = 0;
  for (int64_t li = int64_t(blockIdx.x) * kThreads + threadIdx.x; li < n_local; li += int64_t(gridDim.x) * kThreads) {
    const double y = eval_element(p, base, rank, to_global(p, rank, li, W), W, cr, nullptr, false);
    acc = has ? fold(red, acc, y) : y;
    has = 1;
  }
  s_v[threadIdx.x] = acc;
  s_h[threadIdx.x] = has;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    int h = 0;
    for (int i = 0; i < kThreads; ++i)
      if (s_h[i]) {
        a = h ? fold(red, a, s_v[i]) : s_v[i];
        h = 1;
      }
    block_part[int64_t(li_rank) * gridDim.x + blockIdx.x] = a;
    block_has[int64_t(li_rank) * gridDim.x + blockIdx.x] = h;
  }
}

__global__ void fold_blocks_kernel(const double* block_part, const int* block_has, int nblocks, int red,
                                   double* out) {
  const int r = blockIdx.x;
  if (threadIdx.x != 0) return;
  double a = 0.0;
  int h = 0;
  for (int i = 0; i < nblocks; ++i)
    if (block_has[r * nblocks + i]) {
      a = h ? fold(red, a, block_part[r * nblocks + i]) : block_part[r * nblocks + i];
      h = 1;
    }
  out[r] = a;
}

int local_ranks_of(coconet_ctx* c, int group, LocalRanks* lr) {
  if (!valid_group(c, group)) return set_error(COCONET_ERR_NO_SUCH_RANK, "no such group");
  const coconet_group_s& g = c->groups[size_t(group)];
  std::memset(lr, 0, sizeof(*lr));
  lr->world = g.size;
  if (c->mode == COCONET_MODE_VIRTUAL) {
    for (int i = 0; i < g.size; ++i) {
      lr->base[i] = c->heap[g.first + i];
      lr->rank[i] = i;
    }
  } else {
    if (c->rank < g.first || c->rank >= g.first + g.size)
      return set_error(COCONET_ERR_NO_SUCH_RANK, "this rank is not a member of the group");
    lr->base[0] = c->heap[c->rank];
    lr->rank[0] = c->rank - g.first;
  }
  return COCONET_OK;
}

int validate(const coconet_expr_program* p) {
  if (!p) return set_error(COCONET_ERR_INVALID_INPUT, "null program");
  if (p->n_nodes < 1 || p->n_nodes > COCONET_EXPR_MAX_NODES || p->root < 0 || p->root >= p->n_nodes)
    return set_error(COCONET_ERR_INVALID_INPUT, "bad expression node count/root");
  if (p->n_inputs > COCONET_EXPR_MAX_OPERANDS || p->n_targets > 4 || p->out_ndim > COCONET_EXPR_MAX_DIMS)
    return set_error(COCONET_ERR_INVALID_INPUT, "too many operands");
  for (int i = 0; i < p->n_nodes; ++i) {
    const coconet_expr_node& n = p->nodes[i];
    const bool bin = n.op >= COCONET_OP_ADD && n.op <= COCONET_OP_DIV;
    if ((bin || n.op == COCONET_OP_POW) && (n.a < 0 || n.a >= i || n.b < 0 || n.b >= i))
      return set_error(COCONET_ERR_INVALID_INPUT, "expression nodes must follow their operands");
    if ((n.op == COCONET_OP_SQRT || n.op == COCONET_OP_DROPOUT || n.op == COCONET_OP_UPDATE) && (n.a < 0 || n.a >= i))
      return set_error(COCONET_ERR_INVALID_INPUT, "expression nodes must follow their operands");
    if (n.op == COCONET_OP_INPUT && (n.slot < 0 || n.slot >= p->n_inputs))
      return set_error(COCONET_ERR_INVALID_INPUT, "input slot out of range");
    if (n.op == COCONET_OP_UPDATE && (n.slot < 0 || n.slot >= p->n_targets))
      return set_error(COCONET_ERR_INVALID_INPUT, "update target out of range");
  }
  return COCONET_OK;
}

int small_buffer(coconet_ctx* c, size_t bytes, void** out) {
  if (c->small_bytes < bytes) {
    if (c->small_dev) {
      cudaDeviceSynchronize();
      cudaFree(c->small_dev);
    }
    c->small_dev = nullptr;
    c->small_bytes = 0;
    size_t sz = std::max(bytes, size_t(1) << 20);
    CN_CUDA(cudaMalloc(&c->small_dev, sz));
    c->small_bytes = sz;
  }
  *out = c->small_dev;
  return COCONET_OK;
}

}  // namespace

extern "C" {

int coconet_pointwise(coconet_ctx_t c, int group, const coconet_expr_program* p, const double* rank_consts,
                      const double* reduced, void* stream) {
  if (!c) return set_error(COCONET_ERR_INVALID_INPUT, "null ctx");
  int rc = validate(p);
  if (rc) return rc;
  LocalRanks lr;
  rc = local_ranks_of(c, group, &lr);
  if (rc) return rc;
  const int nl = local_ranks(c, group);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t nc = size_t(nl) * size_t(std::max(0, p->n_rank_consts));
  const size_t nr = size_t(nl) * size_t(std::max(0, p->n_reduce));
  void* buf = nullptr;
  rc = small_buffer(c, (nc + nr + 2) * sizeof(double), &buf);
  if (rc) return rc;
  double* d_consts = static_cast<double*>(buf);
  double* d_red = d_consts + nc + 1;
  if (nc) CN_CUDA(cudaMemcpyAsync(d_consts, rank_consts, nc * sizeof(double), cudaMemcpyHostToDevice, s));
  if (nr) CN_CUDA(cudaMemcpyAsync(d_red, reduced, nr * sizeof(double), cudaMemcpyHostToDevice, s));
  int64_t n = 1;
  for (int d = 0; d < p->out.ndim; ++d) n *= p->out.shape[d];
  const int64_t n_local = p->out_sliced_dim >= 0 ? n / lr.world : n;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n_local + kThreads - 1) / kThreads, 8 * c->sm_count));
  pointwise_kernel<<<dim3(unsigned(blocks), unsigned(nl)), kThreads, 0, s>>>(*p, lr, d_consts, d_red);
  CN_CUDA(cudaGetLastError());
  c->launches++;
  return COCONET_OK;
}

int coconet_pointwise_reduce(coconet_ctx_t c, int group, const coconet_expr_program* p, int node, int red,
                             const double* rank_consts, double* partial, void* stream) {
  (void)node;
  if (!c || !partial) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  int rc = validate(p);
  if (rc) return rc;
  LocalRanks lr;
  rc = local_ranks_of(c, group, &lr);
  if (rc) return rc;
  const int nl = local_ranks(c, group);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t nc = size_t(nl) * size_t(std::max(0, p->n_rank_consts));
  const size_t nb = size_t(nl) * kReduceBlocks;
  void* buf = nullptr;
  rc = small_buffer(c, (nc + 1) * sizeof(double) + nb * (sizeof(double) + sizeof(int)) + nl * sizeof(double) + 64, &buf);
  if (rc) return rc;
  double* d_consts = static_cast<double*>(buf);
  double* d_bp = d_consts + nc + 1;
  double* d_out = d_bp + nb;
  int* d_bh = reinterpret_cast<int*>(d_out + nl);
  if (nc) CN_CUDA(cudaMemcpyAsync(d_consts, rank_consts, nc * sizeof(double), cudaMemcpyHostToDevice, s));
  pointwise_reduce_kernel<<<dim3(kReduceBlocks, unsigned(nl)), kThreads, 0, s>>>(*p, lr, d_consts, red, d_bp, d_bh);
  fold_blocks_kernel<<<nl, 32, 0, s>>>(d_bp, d_bh, kReduceBlocks, red, d_out);
  CN_CUDA(cudaGetLastError());
  c->launches += 2;
  CN_CUDA(cudaMemcpyAsync(partial, d_out, nl * sizeof(double), cudaMemcpyDeviceToHost, s));
  CN_CUDA(cudaStreamSynchronize(s));
  return COCONET_OK;
}

}  // extern "C"
