// Fused data-parallel optimizer step over a tensor list: ReduceScatter +
// Adam/LAMB + AllGather in ONE kernel (paper §3/§6.1, Fig 7b
// "fuse(RS-Opt-AG)"), plus the tensor-list AllReduce it generalises.
//
// Reference semantics being replaced:
//   Engine::exec_data case FusedAllReduce     runtime.hpp:471-516
//     ring_rs_data (fp32, ring order)         runtime.hpp:302-327
//     eval_pointwise of the fused expr         state.hpp:126-193 / expr.hpp:186-222
//     ring_ag_data + gather_decl write-back   runtime.hpp:331-350, 506-510
//   Engine::exec_data case AllReduce           runtime.hpp:384-395 (flat chunks :63-66)
//   scattered_collective                       runtime.hpp:624-675 (no flatten here)
//
// B200 design: one cooperative persistent grid per rank, a WARP per segment
// (a <=1024-element bucket piece, fused_opt.h). TWO_SHOT: each rank pulls
// its own flat chunk of every peer's gradient with 16/8-byte loads (the RS),
// reduces in the reference's ring order in fp32, applies the optimizer in
// registers, and pushes the new parameters into every peer's copy (the AG) —
// no intermediate buffer ever touches HBM. ONE_SHOT pulls everything and keeps
// replicated state (the AR-Opt family). Cross-rank ordering: one flag barrier
// at entry (peers' gradients are ready) and one at exit (peers finished
// reading ours and writing into our parameters).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "fused_opt.h"

namespace cg = cooperative_groups;
using namespace coconet;

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = 2;

struct OptArgs {
  RankSet rs;
  const Seg* segs;
  const int64_t* offs;  // [0,n): g/x heap offsets, [n,2n): p/out heap offsets
  int n_tensors;
  int64_t seg_begin[kMaxRanks + 1];
  int64_t os_begin, os_end;
  int64_t m_off, v_off;
};

// Adam constants in both arithmetics. Double values are exactly what
// eval_expr computes from the f32 decls (Const 1.0 minus double(beta), pow on
// the host like expr.hpp:200).
struct AdamK {
  double b1, b2, cm, cv, bc1, bc2, lr, eps;
  float fb1, fb2, fcm, fcv, frbc1, frbc2, flr, feps;
};

struct LambK {
  double lr;
  float fb1, fb2, fcm, fcv, frbc1, frbc2, feps, fwd;
  const int64_t* csr_ptr;  // per rank: n_tensors+1 entries at csr_begin[r]
  const int64_t* csr_idx;
  double* seg_part;
  int64_t csr_begin[kMaxRanks];
};

__device__ __forceinline__ int rot(int owner, int j, int W) {
  int q = owner + 1 + j;
  q -= (q >= W) ? W : 0;
  q -= (q >= W) ? W : 0;
  return q;
}

// Ring-order reduction of one quad over the group (runtime.hpp:302-305:
// chunk c accumulates x[c+1], x[c+2], ..., x[c]). The loads are issued first
// (W independent 8/16-byte requests), then folded in order.
template <typename T, int RED>
__device__ __forceinline__ void ring_reduce4(char* const* base, int64_t off, int owner, int W,
                                             float acc[4]) {
  float x[kMaxRanks][4];
#pragma unroll
  for (int j = 0; j < kMaxRanks; ++j)
    if (j < W) load4(reinterpret_cast<const T*>(base[rot(owner, j, W)] + off), x[j]);
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i] = x[0][i];
#pragma unroll
  for (int j = 1; j < kMaxRanks; ++j)
    if (j < W) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        // reduce_apply(red, inbox, slot) (types.hpp:76-82): inbox = acc
        if (RED == COCONET_SUM) acc[i] = __fadd_rn(acc[i], x[j][i]);
        else if (RED == COCONET_MAX) acc[i] = acc[i] > x[j][i] ? acc[i] : x[j][i];
        else acc[i] = acc[i] < x[j][i] ? acc[i] : x[j][i];
      }
    }
}

__device__ __forceinline__ void ld4(const float* p, float o[4]) {
  float4 x = *reinterpret_cast<const float4*>(p);
  o[0] = x.x; o[1] = x.y; o[2] = x.z; o[3] = x.w;
}

// Masked quad store: full quads as one vector, partial quads lane by lane.
template <typename T>
__device__ __forceinline__ void st4m(T* p, const float v[4], int lo, int hi) {
  if (lo == 0 && hi == 4) {
    store4(p, v);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i >= lo && i < hi) p[i] = from_f32<T>(v[i]);
  }
}

// Adam element (goldens/adam.json under adam_fused.json):
//   update(p, p - lr*(update(m, m*b1 + cm*g)/bc1) / sqrt(update(v, v*b2 + cv*g*g)/bc2))
// EXACT: IEEE double, explicit _rn intrinsics so nothing is contracted, in
// the parser's association order (json_io.hpp:166-183); Update stores
// float(x) and feeds the unrounded double on (expr.hpp:207-211).
template <int MATH>
__device__ __forceinline__ void adam_elem(float g, float& m, float& v, float& p, const AdamK& k) {
  if (MATH == COCONET_MATH_EXACT) {
    double gd = g;
    double mn = __dadd_rn(__dmul_rn(double(m), k.b1), __dmul_rn(k.cm, gd));
    double vn = __dadd_rn(__dmul_rn(double(v), k.b2), __dmul_rn(__dmul_rn(k.cv, gd), gd));
    double m1 = __ddiv_rn(mn, k.bc1);
    double v1 = __ddiv_rn(vn, k.bc2);
    double den = __dadd_rn(__dsqrt_rn(v1), k.eps);
    double pn = __dsub_rn(double(p), __ddiv_rn(__dmul_rn(k.lr, m1), den));
    m = float(mn);
    v = float(vn);
    p = float(pn);
  } else {
    float mn = fmaf(k.fcm, g, m * k.fb1);
    float vn = fmaf(k.fcv * g, g, v * k.fb2);
    float m1 = mn * k.frbc1;
    float v1 = vn * k.frbc2;
    float upd = __fdividef(k.flr * m1, sqrtf(v1) + k.feps);
    m = mn;
    v = vn;
    p = p - upd;
  }
}

template <typename G, int MATH, bool ONE_SHOT>
__global__ void __launch_bounds__(kThreads) adam_kernel(OptArgs a, AdamK k) {
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int W = rs.world;
  const int me = rs.rank();
  if (!rank_barrier(rs, 0)) return;  // peers' gradients are complete
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sb = ONE_SHOT ? a.os_begin : a.seg_begin[me];
  const int64_t se = ONE_SHOT ? a.os_end : a.seg_begin[me + 1];
  float* m = reinterpret_cast<float*>(s_base[me] + a.m_off);
  float* v = reinterpret_cast<float*>(s_base[me] + a.v_off);
  for (int64_t s = sb + int64_t(blockIdx.x) * kWarps + warp; s < se;
       s += int64_t(gridDim.x) * kWarps) {
    const Seg sg = a.segs[s];
    const int t = meta_tensor(sg.meta), len = meta_len(sg.meta), owner = meta_owner(sg.meta);
    const int64_t goff = a.offs[t], poff = a.offs[a.n_tensors + t];
    const int64_t q0 = sg.toff >> 2, q1 = (sg.toff + len + 3) >> 2;
    for (int64_t qb = q0 + lane; qb < q1; qb += 32 * kUnroll) {
      float g[kUnroll][4], mm[kUnroll][4], vv[kUnroll][4], pp[kUnroll][4];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t q = qb + 32 * u;
        if (q < q1) {
          const int64_t e0 = q << 2;
          const int64_t si = sg.sidx + (e0 - sg.toff);
          ring_reduce4<G, COCONET_SUM>(s_base, goff + e0 * int64_t(sizeof(G)), owner, W, g[u]);
          ld4(m + si, mm[u]);
          ld4(v + si, vv[u]);
          ld4(reinterpret_cast<const float*>(s_base[me] + poff) + e0, pp[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t q = qb + 32 * u;
        if (q < q1) {
          const int64_t e0 = q << 2;
          const int lo = int(max(int64_t(0), sg.toff - e0));
          const int hi = int(min(int64_t(4), sg.toff + len - e0));
          const int64_t si = sg.sidx + (e0 - sg.toff);
#pragma unroll
          for (int i = 0; i < 4; ++i) adam_elem<MATH>(g[u][i], mm[u][i], vv[u][i], pp[u][i], k);
          st4m(m + si, mm[u], lo, hi);
          st4m(v + si, vv[u], lo, hi);
          if (ONE_SHOT) {
            st4m(reinterpret_cast<float*>(s_base[me] + poff) + e0, pp[u], lo, hi);
          } else {
#pragma unroll
            for (int j = 0; j < kMaxRanks; ++j)  // AG push, own copy included
              if (j < W) st4m(reinterpret_cast<float*>(s_base[j] + poff) + e0, pp[u], lo, hi);
          }
        }
      }
    }
  }
  rank_barrier(rs, 1);  // peers done reading our g and writing our p
}

// Tensor-list AllReduce (x -> out). TWO_SHOT = pull-RS of the own chunk +
// push-AG; ONE_SHOT = pull everything, write own copy (out != x).
template <typename T, int RED, bool ONE_SHOT>
__global__ void __launch_bounds__(kThreads) allreduce_kernel(OptArgs a) {
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int W = rs.world;
  const int me = rs.rank();
  if (!rank_barrier(rs, 0)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sb = ONE_SHOT ? a.os_begin : a.seg_begin[me];
  const int64_t se = ONE_SHOT ? a.os_end : a.seg_begin[me + 1];
  for (int64_t s = sb + int64_t(blockIdx.x) * kWarps + warp; s < se;
       s += int64_t(gridDim.x) * kWarps) {
    const Seg sg = a.segs[s];
    const int t = meta_tensor(sg.meta), len = meta_len(sg.meta), owner = meta_owner(sg.meta);
    const int64_t xoff = a.offs[t], ooff = a.offs[a.n_tensors + t];
    const int64_t q0 = sg.toff >> 2, q1 = (sg.toff + len + 3) >> 2;
    for (int64_t qb = q0 + lane; qb < q1; qb += 32 * kUnroll) {
      float acc[kUnroll][4];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t q = qb + 32 * u;
        if (q < q1) ring_reduce4<T, RED>(s_base, xoff + (q << 2) * int64_t(sizeof(T)), owner, W, acc[u]);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t q = qb + 32 * u;
        if (q < q1) {
          const int64_t e0 = q << 2;
          const int lo = int(max(int64_t(0), sg.toff - e0));
          const int hi = int(min(int64_t(4), sg.toff + len - e0));
          if (ONE_SHOT) {
            st4m(reinterpret_cast<T*>(s_base[me] + ooff) + e0, acc[u], lo, hi);
          } else {
#pragma unroll
            for (int j = 0; j < kMaxRanks; ++j)
              if (j < W) st4m(reinterpret_cast<T*>(s_base[j] + ooff) + e0, acc[u], lo, hi);
          }
        }
      }
    }
  }
  rank_barrier(rs, 1);
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// LAMB element direction u = m1/(sqrt(v1)+eps) + wd*p from the stored m, v.
__device__ __forceinline__ float lamb_u(float m, float v, float p, const LambK& k) {
  return __fdividef(m * k.frbc1, sqrtf(v * k.frbc2) + k.feps) + k.fwd * p;
}

// LAMB, two passes inside one cooperative kernel:
//  pass 1: RS pull -> m, v update -> per-segment partial sums of p^2 and u^2
//  grid sync -> per-tensor partials of this rank (fixed segment order, so
//  deterministic) -> pushed into every peer's exchange area -> flag barrier
//  -> totals combined in rank order (state.hpp:163-167)
//  pass 2: trust ratio -> p update -> AG push.
template <typename G>
__global__ void __launch_bounds__(kThreads) lamb_kernel(OptArgs a, LambK k) {
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int W = rs.world;
  const int me = rs.rank();
  // No early return before the grid syncs: a CTA whose barrier timed out
  // skips its work but still arrives, so the grid cannot deadlock.
  const bool ok = rank_barrier(rs, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sb = a.seg_begin[me], se = ok ? a.seg_begin[me + 1] : sb;
  float* m = reinterpret_cast<float*>(s_base[me] + a.m_off);
  float* v = reinterpret_cast<float*>(s_base[me] + a.v_off);
  const int64_t wstride = int64_t(gridDim.x) * kWarps;
  const int64_t wid = int64_t(blockIdx.x) * kWarps + warp;
  // ---- pass 1
  for (int64_t s = sb + wid; s < se; s += wstride) {
    const Seg sg = a.segs[s];
    const int t = meta_tensor(sg.meta), len = meta_len(sg.meta);
    const int64_t goff = a.offs[t], poff = a.offs[a.n_tensors + t];
    const int64_t q0 = sg.toff >> 2, q1 = (sg.toff + len + 3) >> 2;
    double sp = 0.0, su = 0.0;
    for (int64_t qb = q0 + lane; qb < q1; qb += 32 * kUnroll) {
      float g[kUnroll][4], mm[kUnroll][4], vv[kUnroll][4], pp[kUnroll][4];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t q = qb + 32 * u;
        if (q < q1) {
          const int64_t e0 = q << 2;
          const int64_t si = sg.sidx + (e0 - sg.toff);
          ring_reduce4<G, COCONET_SUM>(s_base, goff + e0 * int64_t(sizeof(G)), me, W, g[u]);
          ld4(m + si, mm[u]);
          ld4(v + si, vv[u]);
          ld4(reinterpret_cast<const float*>(s_base[me] + poff) + e0, pp[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t q = qb + 32 * u;
        if (q < q1) {
          const int64_t e0 = q << 2;
          const int lo = int(max(int64_t(0), sg.toff - e0));
          const int hi = int(min(int64_t(4), sg.toff + len - e0));
          const int64_t si = sg.sidx + (e0 - sg.toff);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float mn = fmaf(k.fcm, g[u][i], mm[u][i] * k.fb1);
            float vn = fmaf(k.fcv * g[u][i], g[u][i], vv[u][i] * k.fb2);
            mm[u][i] = mn;
            vv[u][i] = vn;
            if (i >= lo && i < hi) {
              float uu = lamb_u(mn, vn, pp[u][i], k);
              sp += double(pp[u][i]) * double(pp[u][i]);
              su += double(uu) * double(uu);
            }
          }
          st4m(m + si, mm[u], lo, hi);
          st4m(v + si, vv[u], lo, hi);
        }
      }
    }
    sp = warp_sum(sp);
    su = warp_sum(su);
    if (lane == 0) {
      k.seg_part[2 * s] = sp;
      k.seg_part[2 * s + 1] = su;
    }
  }
  __threadfence();
  cg::this_grid().sync();
  // ---- per-tensor partials of this rank -> every peer's exchange slot [me][t]
  const int64_t xch_off = int64_t(kPadBytes) + int64_t(rs.group) * int64_t(kXchBytes / kMaxGroups);
  double* xch_me = reinterpret_cast<double*>(s_base[me] + xch_off);
  for (int64_t t = ok ? wid : a.n_tensors; t < a.n_tensors; t += wstride) {
    const int64_t* ptr = k.csr_ptr + k.csr_begin[me];
    const int64_t b = ptr[t], e = ptr[t + 1];
    double sp = 0.0, su = 0.0;
    for (int64_t i = b + lane; i < e; i += 32) {
      const int64_t s = k.csr_idx[i];
      sp += k.seg_part[2 * s];
      su += k.seg_part[2 * s + 1];
    }
    sp = warp_sum(sp);
    su = warp_sum(su);
    if (lane < W) {
      double* xq = reinterpret_cast<double*>(s_base[lane] + xch_off);
      xq[(int64_t(me) * a.n_tensors + t) * 2] = sp;
      xq[(int64_t(me) * a.n_tensors + t) * 2 + 1] = su;
    }
  }
  __threadfence_system();
  cg::this_grid().sync();
  if (!rank_barrier(rs, 2)) return;
  // ---- pass 2
  for (int64_t s = sb + wid; s < se; s += wstride) {
    const Seg sg = a.segs[s];
    const int t = meta_tensor(sg.meta), len = meta_len(sg.meta);
    const int64_t poff = a.offs[a.n_tensors + t];
    double P = 0.0, U = 0.0;
    for (int q = 0; q < W; ++q) {  // rank order 0..W-1
      P += __ldcg(xch_me + (int64_t(q) * a.n_tensors + t) * 2);
      U += __ldcg(xch_me + (int64_t(q) * a.n_tensors + t) * 2 + 1);
    }
    const float ratio = float((k.lr * sqrt(P)) / sqrt(U));
    const int64_t q0 = sg.toff >> 2, q1 = (sg.toff + len + 3) >> 2;
    for (int64_t qb = q0 + lane; qb < q1; qb += 32 * kUnroll) {
      float mm[kUnroll][4], vv[kUnroll][4], pp[kUnroll][4];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t q = qb + 32 * u;
        if (q < q1) {
          const int64_t e0 = q << 2;
          const int64_t si = sg.sidx + (e0 - sg.toff);
          ld4(m + si, mm[u]);
          ld4(v + si, vv[u]);
          ld4(reinterpret_cast<const float*>(s_base[me] + poff) + e0, pp[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t q = qb + 32 * u;
        if (q < q1) {
          const int64_t e0 = q << 2;
          const int lo = int(max(int64_t(0), sg.toff - e0));
          const int hi = int(min(int64_t(4), sg.toff + len - e0));
          float pn[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) pn[i] = pp[u][i] - ratio * lamb_u(mm[u][i], vv[u][i], pp[u][i], k);
#pragma unroll
          for (int j = 0; j < kMaxRanks; ++j)
            if (j < W) st4m(reinterpret_cast<float*>(s_base[j] + poff) + e0, pn, lo, hi);
        }
      }
    }
  }
  rank_barrier(rs, 1);
}

int fill_args(coconet_tlist* tl, OptArgs* a, const RankSet& rs, int64_t m_off, int64_t v_off) {
  a->rs = rs;
  a->segs = tl->d_segs;
  a->offs = tl->d_offs;
  a->n_tensors = tl->n_tensors;
  for (int r = 0; r <= kMaxRanks; ++r) a->seg_begin[r] = r <= rs.world ? tl->seg_begin[r] : 0;
  a->os_begin = tl->os_begin;
  a->os_end = tl->os_end;
  a->m_off = m_off;
  a->v_off = v_off;
  return COCONET_OK;
}

int64_t max_rank_segs(const coconet_tlist* tl, int W, bool one_shot) {
  if (one_shot) return tl->os_end - tl->os_begin;
  int64_t mx = 0;
  for (int r = 0; r < W; ++r) mx = std::max(mx, tl->seg_begin[r + 1] - tl->seg_begin[r]);
  return mx;
}

int launch_opt(coconet_ctx* c, coconet_tlist* tl, const void* func, void** args, bool one_shot,
               cudaStream_t stream) {
  int W = c->groups[size_t(tl->group)].size;
  int64_t want = (max_rank_segs(tl, W, one_shot) + kWarps - 1) / kWarps;
  int blocks = 0;
  int rc = coop_blocks(c, func, kThreads, 0, tl->group, want, &blocks);
  if (rc) return rc;
  return coop_launch(c, func, dim3(unsigned(blocks), unsigned(local_ranks(c, tl->group))),
                     dim3(kThreads), args, 0, stream);
}

int elem_bytes(int e) { return e == COCONET_F32 ? 4 : 2; }

bool resolve_one_shot(int algo, const coconet_tlist* tl, int W) {
  if (algo == COCONET_ALGO_ONE_SHOT) return true;
  if (algo == COCONET_ALGO_TWO_SHOT) return false;
  // AUTO: the paper's crossover (AR-Opt best up to 2^16 elements,
  // PAPER.md:1558-1565); at W == 1 both are the same local update.
  return W > 1 && tl->total <= (int64_t(1) << 16);
}

template <typename G, int MATH, bool OS>
const void* adam_fn() {
  return reinterpret_cast<const void*>(&adam_kernel<G, MATH, OS>);
}

template <typename G>
const void* adam_pick(int math, bool os) {
  if (math == COCONET_MATH_EXACT) return os ? adam_fn<G, COCONET_MATH_EXACT, true>() : adam_fn<G, COCONET_MATH_EXACT, false>();
  return os ? adam_fn<G, COCONET_MATH_FAST, true>() : adam_fn<G, COCONET_MATH_FAST, false>();
}

template <typename T, int RED>
const void* ar_pick(bool os) {
  return os ? reinterpret_cast<const void*>(&allreduce_kernel<T, RED, true>)
            : reinterpret_cast<const void*>(&allreduce_kernel<T, RED, false>);
}

template <typename T>
const void* ar_pick_red(int red, bool os) {
  if (red == COCONET_MAX) return ar_pick<T, COCONET_MAX>(os);
  if (red == COCONET_MIN) return ar_pick<T, COCONET_MIN>(os);
  return ar_pick<T, COCONET_SUM>(os);
}

int check_state(coconet_ctx* c, const void* ptr, int64_t* off) {
  int rc = heap_offset(c, ptr, off);
  if (rc) return rc;
  if (*off % 16) return set_error(COCONET_ERR_INVALID_INPUT, "optimizer state must be 16-byte aligned");
  return COCONET_OK;
}

}  // namespace

extern "C" {

int coconet_fused_rs_adam_ag(coconet_ctx_t c, coconet_tlist_t tl, const void* const* g, int g_elem,
                             float* const* p, float* m_shard, float* v_shard,
                             const coconet_adam_params* hp, void* stream_) {
  if (!c || !tl || !g || !p || !hp) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  if (tl->ctx != c) return set_error(COCONET_ERR_INVALID_INPUT, "tensor list belongs to another context");
  if (g_elem < COCONET_F32 || g_elem > COCONET_BF16) return set_error(COCONET_ERR_INVALID_INPUT, "bad g elem");
  if (hp->math != COCONET_MATH_EXACT && hp->math != COCONET_MATH_FAST)
    return set_error(COCONET_ERR_INVALID_INPUT, "bad math mode");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int W = c->groups[size_t(tl->group)].size;
  const bool os = resolve_one_shot(hp->algo, tl, W);
  int64_t m_off = 0, v_off = 0;
  int rc = check_state(c, m_shard, &m_off);
  if (!rc) rc = check_state(c, v_shard, &v_off);
  if (!rc) rc = tlist_bind(tl, g, reinterpret_cast<const void* const*>(p), elem_bytes(g_elem), 4, stream);
  if (rc) return rc;
  AdamK k;
  k.b1 = double(hp->beta1);
  k.b2 = double(hp->beta2);
  k.cm = 1.0 - double(hp->beta1);
  k.cv = hp->cv_beta1 ? 1.0 - double(hp->beta1) : 1.0 - double(hp->beta2);
  k.bc1 = 1.0 - std::pow(double(hp->beta1), double(hp->t));
  k.bc2 = 1.0 - std::pow(double(hp->beta2), double(hp->t));
  k.lr = double(hp->lr);
  k.eps = double(hp->eps);
  k.fb1 = hp->beta1;
  k.fb2 = hp->beta2;
  k.fcm = float(k.cm);
  k.fcv = float(k.cv);
  k.frbc1 = float(1.0 / k.bc1);
  k.frbc2 = float(1.0 / k.bc2);
  k.flr = hp->lr;
  k.feps = hp->eps;
  RankSet rs;
  rc = make_rankset(c, tl->group, &rs);
  if (rc) return rc;
  OptArgs a;
  fill_args(tl, &a, rs, m_off, v_off);
  const void* fn = g_elem == COCONET_F32   ? adam_pick<float>(hp->math, os)
                   : g_elem == COCONET_F16 ? adam_pick<__half>(hp->math, os)
                                           : adam_pick<__nv_bfloat16>(hp->math, os);
  void* args[] = {&a, &k};
  return launch_opt(c, tl, fn, args, os, stream);
}

int coconet_fused_rs_lamb_ag(coconet_ctx_t c, coconet_tlist_t tl, const void* const* g, int g_elem,
                             float* const* p, float* m_shard, float* v_shard,
                             const coconet_lamb_params* hp, void* stream_) {
  if (!c || !tl || !g || !p || !hp) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  if (tl->ctx != c) return set_error(COCONET_ERR_INVALID_INPUT, "tensor list belongs to another context");
  if (hp->math != COCONET_MATH_FAST)
    return set_error(COCONET_ERR_UNSUPPORTED,
                     "LAMB runs in FAST math only: its whole-tensor sums cannot reproduce the "
                     "reference's sequential double accumulation bit-for-bit");
  if (size_t(kMaxRanks) * tl->n_tensors * 2 * sizeof(double) > kXchBytes / kMaxGroups)
    return set_error(COCONET_ERR_UNSUPPORTED, "too many tensors for the exchange area");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  int64_t m_off = 0, v_off = 0;
  int rc = check_state(c, m_shard, &m_off);
  if (!rc) rc = check_state(c, v_shard, &v_off);
  if (!rc) rc = tlist_bind(tl, g, reinterpret_cast<const void* const*>(p), elem_bytes(g_elem), 4, stream);
  if (rc) return rc;
  LambK k;
  k.lr = double(hp->lr);
  k.fb1 = hp->beta1;
  k.fb2 = hp->beta2;
  k.fcm = float(1.0 - double(hp->beta1));
  k.fcv = float(1.0 - double(hp->beta2));
  k.frbc1 = float(1.0 / (1.0 - std::pow(double(hp->beta1), double(hp->t))));
  k.frbc2 = float(1.0 / (1.0 - std::pow(double(hp->beta2), double(hp->t))));
  k.feps = hp->eps;
  k.fwd = hp->wd;
  k.csr_ptr = tl->d_csr_ptr;
  k.csr_idx = tl->d_csr_idx;
  k.seg_part = tl->d_seg_part;
  for (int r = 0; r < kMaxRanks; ++r) k.csr_begin[r] = tl->csr_begin[r];
  RankSet rs;
  rc = make_rankset(c, tl->group, &rs);
  if (rc) return rc;
  OptArgs a;
  fill_args(tl, &a, rs, m_off, v_off);
  const void* fn = g_elem == COCONET_F32   ? reinterpret_cast<const void*>(&lamb_kernel<float>)
                   : g_elem == COCONET_F16 ? reinterpret_cast<const void*>(&lamb_kernel<__half>)
                                           : reinterpret_cast<const void*>(&lamb_kernel<__nv_bfloat16>);
  void* args[] = {&a, &k};
  return launch_opt(c, tl, fn, args, false, stream);
}

int coconet_allreduce(coconet_ctx_t c, coconet_tlist_t tl, const void* const* x, void* const* out,
                      int elem, int reducer, int algo, void* stream_) {
  if (!c || !tl || !x || !out) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  if (tl->ctx != c) return set_error(COCONET_ERR_INVALID_INPUT, "tensor list belongs to another context");
  if (elem < COCONET_F32 || elem > COCONET_BF16) return set_error(COCONET_ERR_INVALID_INPUT, "bad elem");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int W = c->groups[size_t(tl->group)].size;
  bool os = resolve_one_shot(algo, tl, W);
  bool in_place = false;
  for (int i = 0; i < tl->n_tensors; ++i) in_place |= (x[i] == out[i]);
  if (in_place) os = false;  // one-shot reads every peer's whole input while writing
  int rc = tlist_bind(tl, x, reinterpret_cast<const void* const*>(out), elem_bytes(elem), elem_bytes(elem), stream);
  if (rc) return rc;
  RankSet rs;
  rc = make_rankset(c, tl->group, &rs);
  if (rc) return rc;
  OptArgs a;
  fill_args(tl, &a, rs, 0, 0);
  const void* fn = elem == COCONET_F32   ? ar_pick_red<float>(reducer, os)
                   : elem == COCONET_F16 ? ar_pick_red<__half>(reducer, os)
                                         : ar_pick_red<__nv_bfloat16>(reducer, os);
  void* args[] = {&a};
  return launch_opt(c, tl, fn, args, os, stream);
}

}  // extern "C"
