// Fused model-parallel and pipeline-parallel epilogues:
//   MP  (goldens/model_parallel.json + schedules/mp_overlap.json):
//       FusedAllReduce{RS(axis 2) -> dropout(layer + b, 0.1) + r -> AG}
//   PP  (goldens/pipeline.json + schedules/pipeline_overlap.json):
//       OverlapGroup{RS (group 0) -> FusedSend{dropout(sum + b, 0.1) + r}
//                    -> AG (group 1)}
//
// Reference semantics: Engine::exec_data FusedAllReduce (runtime.hpp:471-516)
// with axis chunks = column blocks (ChunkSpec axis_chunks :78-85, DistView
// Sliced(d) :62-70), FusedSend (runtime.hpp:439-467), AllGather (:396-414);
// expression semantics eval_expr (expr.hpp:186-222) with the global flat
// element index as the dropout counter (state.hpp:178-181).
//
// B200: one kernel per pattern. MP: rank c pulls column block c of every
// peer's partial sums (ring-order fp32 fold), applies the epilogue in
// registers and pushes the finished block into every peer's output. PP: the
// sender pulls its chunk inside the source stage, applies the epilogue and
// stores it straight into EVERY rank of the next stage — the P2P send and the
// next stage's all-gather become one NVSwitch hop.
#include <cmath>

#include "internal.h"

using namespace coconet;

namespace {

constexpr int kThreads = 256;

struct BdrK {
  double rate, inv_keep;  // rate and 1 - rate, as eval_expr forms them
  float frate_scale;      // 1 / (1 - rate) for FAST
  uint64_t seed, key, thresh;
};

// dropout(x + b, rate, key) + r on one element (expr.hpp:201-205)
template <int MATH>
__device__ __forceinline__ float bdr(float x, float b, float r, uint64_t gi, const BdrK& k) {
  const bool keep = dropout_keep_bits(k.seed, k.key, gi, k.thresh);
  if (MATH == COCONET_MATH_EXACT) {
    double s = __dadd_rn(double(x), double(b));
    double d = keep ? __ddiv_rn(s, k.inv_keep) : 0.0;
    return float(__dadd_rn(d, double(r)));
  } else {
    float d = keep ? (x + b) * k.frate_scale : 0.0f;
    return d + r;
  }
}

template <typename T>
__device__ __forceinline__ void ld4v(const T* p, float o[4], bool vec) {
  if (vec) {
    load4_cg(p, o);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = to_f32(p[i]);
  }
}

struct BdrArgs {
  RankSet rs;
  int64_t x_off, b_off, r_off, out_off;
  int64_t rows, cols, per;  // per = cols / W (column block width)
  int src_ranks;            // PP: union ranks [0, src_ranks) are the senders
  int64_t n;                // PP: elements of the 1-D tensor
};

// 16-byte vectors: V = 16 / sizeof(T) elements kept raw in registers until
// they are folded (the loads of every rank, b and r are all in flight at once).
template <typename T> struct Vec16 {
  static constexpr int V = 16 / int(sizeof(T));
  uint4 raw;
  __device__ __forceinline__ void load_cg(const T* p) { raw = __ldcg(reinterpret_cast<const uint4*>(p)); }
  // streamed once: evict-first
  __device__ __forceinline__ void load_cs(const T* p) { raw = __ldcs(reinterpret_cast<const uint4*>(p)); }
  __device__ __forceinline__ void load(const T* p) { raw = __ldg(reinterpret_cast<const uint4*>(p)); }
  __device__ __forceinline__ float get(int i) const { return to_f32(reinterpret_cast<const T*>(&raw)[i]); }
};

template <typename T>
__device__ __forceinline__ void store16_cs(T* p, const float (&o)[16 / sizeof(T)]) {
  constexpr int V = 16 / int(sizeof(T));
  uint4 raw;
  T* h = reinterpret_cast<T*>(&raw);
#pragma unroll
  for (int i = 0; i < V; ++i) h[i] = from_f32<T>(o[i]);
  __stcs(reinterpret_cast<uint4*>(p), raw);
}
template <typename T>
__device__ __forceinline__ void store16(T* p, const float (&o)[16 / sizeof(T)]) {
  constexpr int V = 16 / int(sizeof(T));
  uint4 raw;
  T* h = reinterpret_cast<T*>(&raw);
#pragma unroll
  for (int i = 0; i < V; ++i) h[i] = from_f32<T>(o[i]);
  *reinterpret_cast<uint4*>(p) = raw;
}

// MP: rank c owns column block c of every row. One 16-byte vector per thread
// per rank; all W + 2 loads issued before the ring-order fold.
template <typename T, int MATH, int WT>
__global__ void __launch_bounds__(kThreads) rs_bdr_ag_kernel(BdrArgs a, BdrK k) {
  constexpr int V = Vec16<T>::V;
  constexpr int kW = WT > 0 ? WT : kMaxRanks;  // group size: compile-time when specialised
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int W = WT > 0 ? WT : rs.world, me = rs.rank();
  if (!edge_barrier(rs, 0)) return;
  const int64_t vpr = a.per / V;  // vectors per row block
  const int64_t nv = a.rows * vpr;
  const T* bb = reinterpret_cast<const T*>(s_base[me] + a.b_off);
  for (int64_t q = int64_t(blockIdx.x) * kThreads + threadIdx.x; q < nv; q += int64_t(gridDim.x) * kThreads) {
    const int64_t row = q / vpr;
    const int64_t col = int64_t(me) * a.per + (q - row * vpr) * V;
    const int64_t gi = row * a.cols + col;
    Vec16<T> x[kW], bv, rv;
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      if (j >= W) break;
      int src = me + 1 + j;
      src -= src >= W ? W : 0;
      src -= src >= W ? W : 0;
      x[j].load_cg(reinterpret_cast<const T*>(s_base[src] + a.x_off) + gi);
    }
    bv.load(bb + col);
    rv.load_cg(reinterpret_cast<const T*>(s_base[me] + a.r_off) + gi);
    float o[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      float acc = x[0].get(i);
#pragma unroll
      for (int j = 1; j < kW; ++j)
        if (j < W) acc = __fadd_rn(acc, x[j].get(i));  // ring order (runtime.hpp:302-305)
      o[i] = bdr<MATH>(acc, bv.get(i), rv.get(i), uint64_t(gi + i), k);
    }
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      if (j >= W) break;
      store16(reinterpret_cast<T*>(s_base[j] + a.out_off) + gi, o);
    }
  }
  edge_barrier(rs, 1);
}

// PP: union ranks [0, S) form the source stage, [S, 2S) the destination.
// Sender i pulls chunk i of `x` from the source ranks (ring order within the
// source stage), applies the epilogue and stores the chunk into `out` of every
// destination rank. V16: 16-byte vectors (8 elements at 16-bit types) when
// every operand and the chunk allow it, else 4-element quads.
template <typename T, int MATH, bool V16, int SS>
__global__ void __launch_bounds__(kThreads) rs_send_ag_kernel(BdrArgs a, BdrK k) {
  constexpr int kS = SS > 0 ? SS : kMaxRanks;  // stage size: compile-time when specialised
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int S = SS > 0 ? SS : a.src_ranks;
  const int U = 2 * S, me = rs.rank();
  if (!edge_barrier(rs, 0)) return;
  if (me < S) {
    const int64_t per = a.n / S;
    if constexpr (V16) {
      // 8 elements per 16-byte vector, kept packed until the fold
      constexpr int VN = Vec16<T>::V;
      const int64_t nv = per / VN;
      for (int64_t q = int64_t(blockIdx.x) * kThreads + threadIdx.x; q < nv; q += int64_t(gridDim.x) * kThreads) {
        const int64_t gi = int64_t(me) * per + q * VN;
        Vec16<T> x[kS], bv, rv;
#pragma unroll
        for (int j = 0; j < kS; ++j) {
          if (j >= S) break;
          int src = me + 1 + j;
          src -= src >= S ? S : 0;
          src -= src >= S ? S : 0;
          x[j].load_cs(reinterpret_cast<const T*>(s_base[src] + a.x_off) + gi);
        }
        bv.load_cs(reinterpret_cast<const T*>(s_base[me] + a.b_off) + gi);
        rv.load_cs(reinterpret_cast<const T*>(s_base[me] + a.r_off) + gi);
        float o[VN];
#pragma unroll
        for (int i = 0; i < VN; ++i) {
          float acc = x[0].get(i);
#pragma unroll
          for (int j = 1; j < kS; ++j)
            if (j < S) acc = __fadd_rn(acc, x[j].get(i));
          o[i] = bdr<MATH>(acc, bv.get(i), rv.get(i), uint64_t(gi + i), k);
        }
#pragma unroll
        for (int j = 0; j < kS; ++j) {
          if (j >= U - S) break;
          store16_cs(reinterpret_cast<T*>(s_base[S + j] + a.out_off) + gi, o);
        }
      }
    } else {
      const int64_t nq = per >> 2;
      for (int64_t q = int64_t(blockIdx.x) * kThreads + threadIdx.x; q < nq; q += int64_t(gridDim.x) * kThreads) {
        const int64_t gi = int64_t(me) * per + q * 4;
        // every source rank's quad, b and r in flight before the fold
        float acc[4], x[kS][4], b4[4], r4[4], o[4];
#pragma unroll
        for (int j = 0; j < kS; ++j) {
          if (j >= S) break;
          int src = me + 1 + j;
          src -= src >= S ? S : 0;
          src -= src >= S ? S : 0;
          load4(reinterpret_cast<const T*>(s_base[src] + a.x_off) + gi, x[j]);
        }
        load4(reinterpret_cast<const T*>(s_base[me] + a.b_off) + gi, b4);
        load4(reinterpret_cast<const T*>(s_base[me] + a.r_off) + gi, r4);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = x[0][i];
#pragma unroll
        for (int j = 1; j < kS; ++j) {
          if (j >= S) break;
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[i] = __fadd_rn(acc[i], x[j][i]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = bdr<MATH>(acc[i], b4[i], r4[i], uint64_t(gi + i), k);
#pragma unroll
        for (int j = 0; j < kS; ++j) {
          if (j >= U - S) break;
          store4(reinterpret_cast<T*>(s_base[S + j] + a.out_off) + gi, o);
        }
      }
    }
  }
  edge_barrier(rs, 1);
}

BdrK make_k(const coconet_bdr_params* hp) {
  BdrK k;
  k.rate = hp->rate;
  k.inv_keep = 1.0 - hp->rate;
  k.frate_scale = float(1.0 / (1.0 - hp->rate));
  k.seed = hp->seed;
  k.key = hp->key;
  // smallest integer t with t * 2^-53 >= rate (exact power-of-two scaling)
  double s = std::ceil(hp->rate * 9007199254740992.0);
  k.thresh = s <= 0 ? 0 : (s >= 9007199254740992.0 ? (uint64_t(1) << 53) : uint64_t(s));
  return k;
}

// EXACT: group size specialised for 2, 4 and 8 (C3 W=8: 151 -> 144 us).
// FAST keeps the generic kernel: specialised, the 8-rank fold measured
// slower (141 -> 166 us) at the same register count.
template <typename T, int MATH>
const void* mp_fn_w(int W) {
  if (MATH == COCONET_MATH_FAST) return reinterpret_cast<const void*>(&rs_bdr_ag_kernel<T, MATH, 0>);
  return W == 8   ? reinterpret_cast<const void*>(&rs_bdr_ag_kernel<T, MATH, 8>)
         : W == 4 ? reinterpret_cast<const void*>(&rs_bdr_ag_kernel<T, MATH, 4>)
         : W == 2 ? reinterpret_cast<const void*>(&rs_bdr_ag_kernel<T, MATH, 2>)
                  : reinterpret_cast<const void*>(&rs_bdr_ag_kernel<T, MATH, 0>);
}

template <int MATH>
const void* mp_fn(int elem, int W) {
  switch (elem) {
    case COCONET_F16: return mp_fn_w<__half, MATH>(W);
    case COCONET_BF16: return mp_fn_w<__nv_bfloat16, MATH>(W);
    default: return mp_fn_w<float, MATH>(W);
  }
}

// stage size specialised for 2 and 4 (the paper's 2 x 4 boundary), generic otherwise
template <typename T, int MATH, bool V16>
const void* pp_fn_s(int S) {
  return S == 4   ? reinterpret_cast<const void*>(&rs_send_ag_kernel<T, MATH, V16, 4>)
         : S == 2 ? reinterpret_cast<const void*>(&rs_send_ag_kernel<T, MATH, V16, 2>)
                  : reinterpret_cast<const void*>(&rs_send_ag_kernel<T, MATH, V16, 0>);
}

template <int MATH>
const void* pp_fn(int elem, bool v16, int S) {
  switch (elem) {
    case COCONET_F16: return v16 ? pp_fn_s<__half, MATH, true>(S) : pp_fn_s<__half, MATH, false>(S);
    case COCONET_BF16:
      return v16 ? pp_fn_s<__nv_bfloat16, MATH, true>(S) : pp_fn_s<__nv_bfloat16, MATH, false>(S);
    default: return pp_fn_s<float, MATH, false>(S);  // fp32 quads are 16 bytes already
  }
}

int esz(int e) { return e == COCONET_F32 ? 4 : 2; }

int offsets(coconet_ctx* c, const void* x, const void* b, const void* r, const void* out, int elem,
            BdrArgs* a) {
  int rc = heap_offset(c, x, &a->x_off);
  if (!rc) rc = heap_offset(c, b, &a->b_off);
  if (!rc) rc = heap_offset(c, r, &a->r_off);
  if (!rc) rc = heap_offset(c, out, &a->out_off);
  if (rc) return rc;
  if ((a->x_off | a->b_off | a->r_off | a->out_off) % (4 * esz(elem)))
    return set_error(COCONET_ERR_INVALID_INPUT, "operands must be aligned to 4 elements");
  return COCONET_OK;
}

// group covering [first, first+size): an existing one, or a new one
int union_group(coconet_ctx* c, int first, int size, int* g) {
  for (size_t i = 0; i < c->groups.size(); ++i)
    if (c->groups[i].first == first && c->groups[i].size == size) {
      *g = int(i);
      return COCONET_OK;
    }
  return coconet_group_create(c, first, size, g);
}

}  // namespace

extern "C" {

int coconet_fused_rs_bdr_ag(coconet_ctx_t c, int group, const void* x, const void* b, const void* r,
                            void* out, int elem, int64_t rows, int64_t cols,
                            const coconet_bdr_params* hp, void* stream) {
  if (!c || !hp) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  if (!valid_group(c, group)) return set_error(COCONET_ERR_NO_SUCH_RANK, "no such group");
  if (elem < COCONET_F32 || elem > COCONET_BF16) return set_error(COCONET_ERR_INVALID_INPUT, "bad elem");
  const int W = c->groups[size_t(group)].size;
  if (cols % W)
    return set_error(COCONET_ERR_DIVISIBILITY, "extent " + std::to_string(cols) + " over " + std::to_string(W) + " ranks");
  if ((cols / W) % (16 / esz(elem)))
    return set_error(COCONET_ERR_UNSUPPORTED, "column block must be a multiple of 16 bytes");
  BdrArgs a{};
  int rc = offsets(c, x, b, r, out, elem, &a);
  if (rc) return rc;
  if ((a.x_off | a.b_off | a.r_off | a.out_off | (cols * esz(elem))) % 16)
    return set_error(COCONET_ERR_INVALID_INPUT, "operands and rows must be 16-byte aligned");
  a.rows = rows;
  a.cols = cols;
  a.per = cols / W;
  BdrK k = make_k(hp);
  const void* fn = hp->math == COCONET_MATH_EXACT ? mp_fn<COCONET_MATH_EXACT>(elem, W)
                                                  : mp_fn<COCONET_MATH_FAST>(elem, W);
  int blocks = 0;
  rc = coop_blocks(c, fn, kThreads, 0, group, (rows * (a.per / (16 / esz(elem))) + kThreads - 1) / kThreads, &blocks);
  if (!rc) rc = make_rankset(c, group, &a.rs);
  if (rc) return rc;
  void* args[] = {&a, &k};
  return coop_launch(c, fn, dim3(unsigned(blocks), unsigned(local_ranks(c, group))), dim3(kThreads), args, 0,
                     static_cast<cudaStream_t>(stream));
}

int coconet_rs_fused_send_ag(coconet_ctx_t c, int src_group, int dst_group, const void* x, const void* b,
                             const void* r, void* out, int elem, int64_t n, const coconet_bdr_params* hp,
                             void* stream) {
  if (!c || !hp) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  if (!valid_group(c, src_group) || !valid_group(c, dst_group))
    return set_error(COCONET_ERR_NO_SUCH_RANK, "no such group");
  const coconet_group_s gs = c->groups[size_t(src_group)], gd = c->groups[size_t(dst_group)];
  // FusedSend: "peer group sizes differ" (runtime.hpp:448)
  if (gs.size != gd.size) return set_error(COCONET_ERR_NO_SUCH_RANK, "peer group sizes differ");
  if (gd.first != gs.first + gs.size)
    return set_error(COCONET_ERR_UNSUPPORTED, "the destination stage must follow the source stage");
  if (n % gs.size) return set_error(COCONET_ERR_DIVISIBILITY, "extent does not divide over the stage");
  if ((n / gs.size) % 4) return set_error(COCONET_ERR_UNSUPPORTED, "chunk must be a multiple of 4 elements");
  BdrArgs a{};
  int rc = offsets(c, x, b, r, out, elem, &a);
  if (rc) return rc;
  a.n = n;
  a.src_ranks = gs.size;
  int ug = 0;
  rc = union_group(c, gs.first, gs.size + gd.size, &ug);
  if (rc) return rc;
  BdrK k = make_k(hp);
  // 16-bit types: 8-element vectors when every operand is 16-byte aligned and
  // the chunk is a multiple of 8 elements
  const bool v16 = elem != COCONET_F32 && (n / gs.size) % 8 == 0 &&
                   ((a.x_off | a.b_off | a.r_off | a.out_off) % 16) == 0;
  const void* fn =
      hp->math == COCONET_MATH_EXACT ? pp_fn<COCONET_MATH_EXACT>(elem, v16, gs.size)
                                     : pp_fn<COCONET_MATH_FAST>(elem, v16, gs.size);
  const int vn = v16 ? 8 : 4;
  // Only the source stage computes. VIRTUAL: the grid covers the S sender
  // ranks only (blockIdx.y = union rank < S), so every resident CTA moves
  // data (the destination ranks' CTAs would only meet no-op edge barriers);
  // DISTRIBUTED: every process launches its own rank (receivers take part in
  // the entry/exit barriers).
  int blocks = 0;
  rc = coop_blocks(c, fn, kThreads, 0, src_group, (n / gs.size / vn + kThreads - 1) / kThreads, &blocks);
  if (!rc) rc = make_rankset(c, ug, &a.rs);
  if (rc) return rc;
  void* args[] = {&a, &k};
  return coop_launch(c, fn, dim3(unsigned(blocks), unsigned(local_ranks(c, src_group))), dim3(kThreads), args, 0,
                     static_cast<cudaStream_t>(stream));
}

}  // extern "C"
