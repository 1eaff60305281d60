// Axis-sliced ReduceScatter / AllGather of one tensor over a group, and the
// rooted Reduce / Broadcast.
//
// Reference: Engine::run_reduce_scatter (runtime.hpp:352-363) and the
// AllGather case (runtime.hpp:396-414) with ChunkSpec::axis_chunks
// (runtime.hpp:78-85): chunk c is rank c's DistView slice (view.hpp:62-70),
// i.e. `before` runs of `per*stride_d` contiguous elements. exec_gather_decl
// (runtime.hpp:529-557) is the in-place AllGather of an updated decl.
//
// B200: pull-RS (each rank reads its slice from every peer over NVLink and
// folds in ring order) and push-AG (each rank stores its slice into every
// peer); quads of 4 elements when the contiguous runs allow, flag barriers at
// entry/exit as in fused_opt.cu.
//
// Reduce (runtime.hpp:415-428): the root pulls every rank's tensor and folds
// in RANK order 0..G-1 in fp32 (acc = x_0; acc = reduce_apply(acc, x_r)),
// exactly as the Engine does; other ranks' outputs are zero (Local layout,
// meaningful on the root only, program.hpp:315-321). Broadcast (:429-436):
// every rank pulls the root's tensor (the root's NVLink egress is (G-1)*N,
// as in the reference's byte count).
#include <algorithm>
#include <string>

#include "internal.h"

using namespace coconet;

namespace {

constexpr int kThreads = 256;

struct AxisArgs {
  RankSet rs;
  int64_t x_off, out_off;  // heap offsets
  int64_t n_local;         // slice elements per rank
  int64_t run;             // per * stride_d (contiguous elements per run)
  int64_t global_run;      // G_d * stride_d
  int reducer;
  int in_place;            // AG from `out` itself (gather_decl)
};

__device__ __forceinline__ int64_t slice_to_global(const AxisArgs& a, int rank, int64_t li) {
  const int64_t before = li / a.run;
  return before * a.global_run + int64_t(rank) * a.run + (li - before * a.run);
}

template <typename T, int RED>
__device__ __forceinline__ float fold(float acc, float x) {
  if (RED == COCONET_SUM) return __fadd_rn(acc, x);
  if (RED == COCONET_MAX) return acc > x ? acc : x;
  return acc < x ? acc : x;
}

// RS: out_r[li] = ring-order fold over q of x_q[to_global(r, li)].
struct RootArgs {
  RankSet rs;
  int64_t x_off, out_off, n;
  int root;
};

// Reduce: the root folds x over ranks 0..G-1; after the exit barrier (the
// root is done reading every x) the other ranks zero their output, so x may
// alias out.
template <typename T, int RED, int VEC>
__global__ void __launch_bounds__(kThreads) reduce_kernel(RootArgs a) {
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int W = rs.world, me = rs.rank();
  if (!edge_barrier(rs, 0)) return;
  const int64_t nq = a.n / VEC;
  const int64_t st = int64_t(gridDim.x) * kThreads;
  if (me == a.root) {
    T* out = reinterpret_cast<T*>(s_base[me] + a.out_off);
    for (int64_t q = int64_t(blockIdx.x) * kThreads + threadIdx.x; q < nq; q += st) {
      float acc[VEC], x[VEC];
#pragma unroll
      for (int j = 0; j < kMaxRanks; ++j) {
        if (j >= W) break;
        const T* xs = reinterpret_cast<const T*>(s_base[j] + a.x_off) + q * VEC;
        if (VEC == 4) load4_cg(xs, x);
        else x[0] = to_f32(xs[0]);
#pragma unroll
        for (int i = 0; i < VEC; ++i) acc[i] = j == 0 ? x[i] : fold<T, RED>(acc[i], x[i]);
      }
      if (VEC == 4) store4(out + q * VEC, acc);
      else out[q] = from_f32<T>(acc[0]);
    }
  }
  // pairwise with the root's CTA of the same index: this CTA then zeroes
  // exactly the vectors that CTA read
  if (!rank_barrier(rs, 1)) return;
  if (me != a.root) {
    T* out = reinterpret_cast<T*>(s_base[me] + a.out_off);
    for (int64_t q = int64_t(blockIdx.x) * kThreads + threadIdx.x; q < nq; q += st)
#pragma unroll
      for (int i = 0; i < VEC; ++i) out[q * VEC + i] = from_f32<T>(0.f);
  }
}

// Broadcast: every rank copies the root's x into its out.
template <typename T, int VEC>
__global__ void __launch_bounds__(kThreads) bcast_kernel(RootArgs a) {
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int me = rs.rank();
  if (!edge_barrier(rs, 0)) return;
  const bool same = me == a.root && a.x_off == a.out_off;
  if (!same) {
    const T* src = reinterpret_cast<const T*>(s_base[a.root] + a.x_off);
    T* out = reinterpret_cast<T*>(s_base[me] + a.out_off);
    const int64_t nq = a.n / VEC;
    for (int64_t q = int64_t(blockIdx.x) * kThreads + threadIdx.x; q < nq; q += int64_t(gridDim.x) * kThreads) {
      if (VEC == 4) {
        float x[4];
        load4_cg(src + q * 4, x);
        store4(out + q * 4, x);
      } else {
        out[q] = src[q];
      }
    }
  }
  edge_barrier(rs, 1);  // nobody overwrites the root's x while peers still read it (across processes)
}

// Send (runtime.hpp:439-470): group rank r of the source stage stores its n
// local elements into group rank r of the destination stage (a push over
// NVLink). Launched over the rank interval covering both stages: the entry
// barrier orders the push after the destination's previous readers, the exit
// barrier makes it visible before the destination's next kernel.
struct SendArgs {
  RankSet rs;
  int64_t x_off, out_off, n;
  int src_first, dst_first, size;  // union-relative first ranks, stage size
};

template <typename T, int VEC>
__global__ void __launch_bounds__(kThreads) send_kernel(SendArgs a) {
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int me = rs.rank();
  if (!edge_barrier(rs, 0)) return;
  const int sr = me - a.src_first;
  if (sr >= 0 && sr < a.size) {
    const T* src = reinterpret_cast<const T*>(s_base[me] + a.x_off);
    T* dst = reinterpret_cast<T*>(s_base[a.dst_first + sr] + a.out_off);
    const int64_t nq = a.n / VEC;
    for (int64_t q = int64_t(blockIdx.x) * kThreads + threadIdx.x; q < nq; q += int64_t(gridDim.x) * kThreads) {
      if (VEC == 4) {
        float x[4];
        load4_cg(src + q * 4, x);
        store4(dst + q * 4, x);
      } else {
        dst[q] = src[q];
      }
    }
  }
  edge_barrier(rs, 1);
}

// Element type conversion of a plain device array (the 16-bit staging of
// fp32-stored decls for the tcgen05 MatMul; not collective).
template <typename S, typename D>
__global__ void __launch_bounds__(kThreads) convert_kernel(const S* src, D* dst, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * kThreads + threadIdx.x; i < n; i += int64_t(gridDim.x) * kThreads)
    dst[i] = from_f32<D>(to_f32(src[i]));
}

template <typename T, int RED, int VEC>
__global__ void __launch_bounds__(kThreads) rs_kernel(AxisArgs a) {
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int W = rs.world, me = rs.rank();
  if (!edge_barrier(rs, 0)) return;
  T* out = reinterpret_cast<T*>(s_base[me] + a.out_off);
  const int64_t nq = a.n_local / VEC;
  for (int64_t q = int64_t(blockIdx.x) * kThreads + threadIdx.x; q < nq; q += int64_t(gridDim.x) * kThreads) {
    const int64_t li = q * VEC;
    const int64_t gi = slice_to_global(a, me, li);
    float acc[VEC], x[VEC];
#pragma unroll
    for (int j = 0; j < kMaxRanks; ++j) {
      if (j >= W) break;
      int src = me + 1 + j;
      src -= src >= W ? W : 0;
      src -= src >= W ? W : 0;
      const T* xs = reinterpret_cast<const T*>(s_base[src] + a.x_off) + gi;
      if (VEC == 4) load4(xs, x);
      else x[0] = to_f32(xs[0]);
#pragma unroll
      for (int i = 0; i < VEC; ++i) acc[i] = j == 0 ? x[i] : fold<T, RED>(acc[i], x[i]);
    }
    if (VEC == 4) store4(out + li, acc);
    else out[li] = from_f32<T>(acc[0]);
  }
  edge_barrier(rs, 1);
}

// AG: out_q[to_global(r, li)] = x_r[li] for every q (push). in_place: the
// source is out_r's own region.
template <typename T, int VEC>
__global__ void __launch_bounds__(kThreads) ag_kernel(AxisArgs a) {
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int W = rs.world, me = rs.rank();
  if (!edge_barrier(rs, 0)) return;
  const int64_t nq = a.n_local / VEC;
  for (int64_t q = int64_t(blockIdx.x) * kThreads + threadIdx.x; q < nq; q += int64_t(gridDim.x) * kThreads) {
    const int64_t li = q * VEC;
    const int64_t gi = slice_to_global(a, me, li);
    const T* src = a.in_place ? reinterpret_cast<const T*>(s_base[me] + a.out_off) + gi
                              : reinterpret_cast<const T*>(s_base[me] + a.x_off) + li;
    float x[VEC];
    if (VEC == 4) load4_cg(src, x);
    else x[0] = to_f32(src[0]);
#pragma unroll
    for (int j = 0; j < kMaxRanks; ++j) {
      if (j >= W) break;
      if (a.in_place && j == me) continue;
      T* dst = reinterpret_cast<T*>(s_base[j] + a.out_off) + gi;
      if (VEC == 4) store4(dst, x);
      else dst[0] = from_f32<T>(x[0]);
    }
  }
  edge_barrier(rs, 1);
}

template <typename T, int VEC>
const void* rs_fn(int red) {
  if (red == COCONET_MAX) return reinterpret_cast<const void*>(&rs_kernel<T, COCONET_MAX, VEC>);
  if (red == COCONET_MIN) return reinterpret_cast<const void*>(&rs_kernel<T, COCONET_MIN, VEC>);
  return reinterpret_cast<const void*>(&rs_kernel<T, COCONET_SUM, VEC>);
}

template <typename T>
const void* rs_pick(int red, bool vec) { return vec ? rs_fn<T, 4>(red) : rs_fn<T, 1>(red); }

template <typename T>
const void* ag_pick(bool vec) {
  return vec ? reinterpret_cast<const void*>(&ag_kernel<T, 4>) : reinterpret_cast<const void*>(&ag_kernel<T, 1>);
}

int setup(coconet_ctx* c, int group, int ndim, const int64_t* shape, int axis, int elem, AxisArgs* a,
          bool* vec) {
  if (!valid_group(c, group)) return set_error(COCONET_ERR_NO_SUCH_RANK, "no such group");
  if (ndim < 1 || ndim > 8 || !shape) return set_error(COCONET_ERR_INVALID_INPUT, "bad shape");
  if (axis < 0) axis = ndim - 1;
  if (axis >= ndim) return set_error(COCONET_ERR_INVALID_INPUT, "axis out of range");
  const int W = c->groups[size_t(group)].size;
  if (shape[axis] % W)
    return set_error(COCONET_ERR_DIVISIBILITY,
                     "extent " + std::to_string(shape[axis]) + " over " + std::to_string(W) + " ranks");
  if (elem < COCONET_F32 || elem > COCONET_BF16) return set_error(COCONET_ERR_INVALID_INPUT, "bad elem");
  int64_t total = 1, stride = 1;
  for (int i = 0; i < ndim; ++i) total *= shape[i];
  for (int i = axis + 1; i < ndim; ++i) stride *= shape[i];
  a->run = shape[axis] / W * stride;
  a->global_run = shape[axis] * stride;
  a->n_local = total / W;
  *vec = (a->run % 4) == 0;
  return COCONET_OK;
}

int launch(coconet_ctx* c, int group, const void* fn, AxisArgs* a, bool vec, cudaStream_t s) {
  int64_t units = vec ? a->n_local / 4 : a->n_local;
  int blocks = 0;
  int rc = coop_blocks(c, fn, kThreads, 0, group, (units + kThreads - 1) / kThreads, &blocks);
  if (rc) return rc;
  rc = make_rankset(c, group, &a->rs);
  if (rc) return rc;
  void* args[] = {a};
  return coop_launch(c, fn, dim3(unsigned(blocks), unsigned(local_ranks(c, group))), dim3(kThreads), args, 0, s);
}

int elem_size(int e) { return e == COCONET_F32 ? 4 : 2; }

template <typename T, int VEC>
const void* reduce_fn(int red) {
  if (red == COCONET_MAX) return reinterpret_cast<const void*>(&reduce_kernel<T, COCONET_MAX, VEC>);
  if (red == COCONET_MIN) return reinterpret_cast<const void*>(&reduce_kernel<T, COCONET_MIN, VEC>);
  return reinterpret_cast<const void*>(&reduce_kernel<T, COCONET_SUM, VEC>);
}

template <typename T>
const void* reduce_pick(int red, bool vec) { return vec ? reduce_fn<T, 4>(red) : reduce_fn<T, 1>(red); }

template <typename T>
const void* bcast_pick(bool vec) {
  return vec ? reinterpret_cast<const void*>(&bcast_kernel<T, 4>) : reinterpret_cast<const void*>(&bcast_kernel<T, 1>);
}

int rooted(coconet_ctx* c, int group, const void* x, void* out, int elem, int64_t n, int root, bool is_reduce,
           int reducer, cudaStream_t s) {
  if (!c || !x || !out) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  if (!valid_group(c, group)) return set_error(COCONET_ERR_NO_SUCH_RANK, "no such group");
  const int W = c->groups[size_t(group)].size;
  if (root < 0 || root >= W) return set_error(COCONET_ERR_NO_SUCH_RANK, "root " + std::to_string(root) + " out of range");
  if (n < 0) return set_error(COCONET_ERR_SHAPE_MISMATCH, "negative element count");
  if (elem < COCONET_F32 || elem > COCONET_BF16) return set_error(COCONET_ERR_INVALID_INPUT, "bad elem");
  if (is_reduce && (reducer < COCONET_SUM || reducer > COCONET_MIN))
    return set_error(COCONET_ERR_INVALID_INPUT, "bad reducer");
  RootArgs a{};
  int rc = heap_offset(c, x, &a.x_off);
  if (!rc) rc = heap_offset(c, out, &a.out_off);
  if (rc) return rc;
  a.n = n;
  a.root = root;
  const bool vec = n % 4 == 0 && (a.x_off | a.out_off) % (4 * elem_size(elem)) == 0;
  const void* fn = is_reduce ? (elem == COCONET_F32   ? reduce_pick<float>(reducer, vec)
                                : elem == COCONET_F16 ? reduce_pick<__half>(reducer, vec)
                                                      : reduce_pick<__nv_bfloat16>(reducer, vec))
                             : (elem == COCONET_F32   ? bcast_pick<float>(vec)
                                : elem == COCONET_F16 ? bcast_pick<__half>(vec)
                                                      : bcast_pick<__nv_bfloat16>(vec));
  const int64_t units = vec ? n / 4 : n;
  int blocks = 0;
  rc = coop_blocks(c, fn, kThreads, 0, group, std::max<int64_t>(1, (units + kThreads - 1) / kThreads), &blocks);
  if (rc) return rc;
  rc = make_rankset(c, group, &a.rs);
  if (rc) return rc;
  void* args[] = {&a};
  return coop_launch(c, fn, dim3(unsigned(blocks), unsigned(local_ranks(c, group))), dim3(kThreads), args, 0, s);
}

}  // namespace

extern "C" {

int coconet_reduce_scatter(coconet_ctx_t c, int group, const void* x, void* out, int elem, int reducer,
                           int ndim, const int64_t* shape, int axis, void* stream) {
  if (!c || !x || !out) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  AxisArgs a{};
  bool vec = false;
  int rc = setup(c, group, ndim, shape, axis, elem, &a, &vec);
  if (!rc) rc = heap_offset(c, x, &a.x_off);
  if (!rc) rc = heap_offset(c, out, &a.out_off);
  if (rc) return rc;
  if (vec && ((a.x_off | a.out_off) % (4 * elem_size(elem)))) vec = false;
  a.reducer = reducer;
  const void* fn = elem == COCONET_F32   ? rs_pick<float>(reducer, vec)
                   : elem == COCONET_F16 ? rs_pick<__half>(reducer, vec)
                                         : rs_pick<__nv_bfloat16>(reducer, vec);
  return launch(c, group, fn, &a, vec, static_cast<cudaStream_t>(stream));
}

int coconet_all_gather(coconet_ctx_t c, int group, const void* x, void* out, int elem, int ndim,
                       const int64_t* shape, int axis, void* stream) {
  if (!c || !out) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  AxisArgs a{};
  bool vec = false;
  int rc = setup(c, group, ndim, shape, axis, elem, &a, &vec);
  if (!rc && x) rc = heap_offset(c, x, &a.x_off);
  if (!rc) rc = heap_offset(c, out, &a.out_off);
  if (rc) return rc;
  a.in_place = x == nullptr;
  if (vec && ((a.x_off | a.out_off) % (4 * elem_size(elem)))) vec = false;
  const void* fn = elem == COCONET_F32   ? ag_pick<float>(vec)
                   : elem == COCONET_F16 ? ag_pick<__half>(vec)
                                         : ag_pick<__nv_bfloat16>(vec);
  return launch(c, group, fn, &a, vec, static_cast<cudaStream_t>(stream));
}

int coconet_send(coconet_ctx_t c, int src_group, int dst_group, const void* x, void* out, int elem, int64_t n,
                 void* stream) {
  if (!c || !x || !out) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  if (!valid_group(c, src_group) || !valid_group(c, dst_group))
    return set_error(COCONET_ERR_NO_SUCH_RANK, "no such group");
  const coconet_group_s gs = c->groups[size_t(src_group)], gd = c->groups[size_t(dst_group)];
  if (gs.size != gd.size) return set_error(COCONET_ERR_NO_SUCH_RANK, "peer group sizes differ");  // runtime.hpp:448
  if (n < 0) return set_error(COCONET_ERR_SHAPE_MISMATCH, "negative element count");
  if (elem < COCONET_F32 || elem > COCONET_BF16) return set_error(COCONET_ERR_INVALID_INPUT, "bad elem");
  const int first = std::min(gs.first, gd.first);
  const int end = std::max(gs.first + gs.size, gd.first + gd.size);
  int ug = -1;
  for (size_t i = 0; i < c->groups.size(); ++i)
    if (c->groups[i].first == first && c->groups[i].size == end - first) ug = int(i);
  if (ug < 0) {
    int rc = coconet_group_create(c, first, end - first, &ug);
    if (rc) return rc;
  }
  SendArgs a{};
  int rc = heap_offset(c, x, &a.x_off);
  if (!rc) rc = heap_offset(c, out, &a.out_off);
  if (rc) return rc;
  a.n = n;
  a.src_first = gs.first - first;
  a.dst_first = gd.first - first;
  a.size = gs.size;
  const bool vec = n % 4 == 0 && (a.x_off | a.out_off) % (4 * elem_size(elem)) == 0;
  auto pick = [&](auto tag) -> const void* {
    using T = decltype(tag);
    return vec ? reinterpret_cast<const void*>(&send_kernel<T, 4>) : reinterpret_cast<const void*>(&send_kernel<T, 1>);
  };
  const void* fn = elem == COCONET_F32 ? pick(float{}) : elem == COCONET_F16 ? pick(__half{}) : pick(__nv_bfloat16{});
  const int64_t units = vec ? n / 4 : n;
  int blocks = 0;
  rc = coop_blocks(c, fn, kThreads, 0, ug, std::max<int64_t>(1, (units + kThreads - 1) / kThreads), &blocks);
  if (!rc) rc = make_rankset(c, ug, &a.rs);
  if (rc) return rc;
  void* args[] = {&a};
  return coop_launch(c, fn, dim3(unsigned(blocks), unsigned(local_ranks(c, ug))), dim3(kThreads), args, 0,
                     static_cast<cudaStream_t>(stream));
}

int coconet_convert(coconet_ctx_t c, const void* src, int src_elem, void* dst, int dst_elem, int64_t n,
                    void* stream) {
  if (!c || (n > 0 && (!src || !dst))) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  if (src_elem < COCONET_F32 || src_elem > COCONET_BF16 || dst_elem < COCONET_F32 || dst_elem > COCONET_BF16)
    return set_error(COCONET_ERR_INVALID_INPUT, "bad elem");
  if (n <= 0) return COCONET_OK;
  const unsigned blocks = unsigned(std::min<int64_t>((n + kThreads - 1) / kThreads, int64_t(c->sm_count) * 8));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto go = [&](auto ts) {
    using S = decltype(ts);
    auto to = [&](auto td) {
      using D = decltype(td);
      convert_kernel<S, D><<<blocks, kThreads, 0, s>>>(static_cast<const S*>(src), static_cast<D*>(dst), n);
    };
    if (dst_elem == COCONET_F32) to(float{});
    else if (dst_elem == COCONET_F16) to(__half{});
    else to(__nv_bfloat16{});
  };
  if (src_elem == COCONET_F32) go(float{});
  else if (src_elem == COCONET_F16) go(__half{});
  else go(__nv_bfloat16{});
  CN_CUDA(cudaGetLastError());
  c->launches++;
  return COCONET_OK;
}

int coconet_reduce(coconet_ctx_t c, int group, const void* x, void* out, int elem, int reducer, int64_t n,
                   int root, void* stream) {
  return rooted(c, group, x, out, elem, n, root, true, reducer, static_cast<cudaStream_t>(stream));
}

int coconet_broadcast(coconet_ctx_t c, int group, const void* x, void* out, int elem, int64_t n, int root,
                      void* stream) {
  return rooted(c, group, x, out, elem, n, root, false, COCONET_SUM, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
