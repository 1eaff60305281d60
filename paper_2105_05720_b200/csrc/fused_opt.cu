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
//
// Latency hiding (the kernels are HBM/NVLink streams): the group size is a
// template parameter (register arrays sized exactly), segment descriptors are
// prefetched two segments ahead (the descriptor -> tensor-offset -> data
// chain would otherwise be exposed per segment), and each lane keeps UNROLL
// quads' loads in flight before consuming any.
#include <cooperative_groups.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <cmath>

#include "fused_opt.h"
#include "pipeline.cuh"

namespace cg = cooperative_groups;
using namespace coconet;

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct OptArgs {
  RankSet rs;
  const Seg* segs;
  const int64_t* offs;  // [0,n): g/x heap offsets, [n,2n): p/out heap offsets
  int n_tensors;
  int64_t seg_begin[kMaxRanks + 1];
  int64_t os_begin, os_end;
  int64_t m_off, v_off;
  int parts;  // adam_kernel: quad ranges per segment (1 = whole segments)
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
  // EXACT: the double constants eval_expr forms from the f32 decls
  double b1, b2, c1, c2, bc1, bc2, eps, wd;
  int guard;  // trust_ratio(): lr when a norm is 0 (apex/NVLAMB) instead of the raw formula
  const int64_t* csr_ptr;  // per rank: n_tensors+1 entries at csr_begin[r]
  const int64_t* csr_idx;
  double* seg_part;
  int64_t csr_begin[kMaxRanks];
};

// Compile-time group size (WT > 0) or runtime W <= kMaxRanks (WT == 0).
template <int WT> struct Ranks {
  static constexpr int kMax = WT > 0 ? WT : kMaxRanks;
  __device__ __forceinline__ static bool has(int j, int W) { return WT > 0 ? true : j < W; }
};

template <int WT>
__device__ __forceinline__ int rot(int owner, int j, int W) {
  const int w = WT > 0 ? WT : W;
  int q = owner + 1 + j;
  q -= (q >= w) ? w : 0;
  q -= (q >= w) ? w : 0;
  return q;
}

// Ring-order reduction of one quad over the group (runtime.hpp:302-305:
// chunk c accumulates x[c+1], x[c+2], ..., x[c]). The loads are issued first
// (W independent 8/16-byte requests), then folded in order.
template <typename T, int RED, int WT>
__device__ __forceinline__ void ring_load4(char* const* base, int64_t off, int owner, int W,
                                           float x[][4]) {
#pragma unroll
  for (int j = 0; j < Ranks<WT>::kMax; ++j)
    if (Ranks<WT>::has(j, W)) load4(reinterpret_cast<const T*>(base[rot<WT>(owner, j, W)] + off), x[j]);
}

template <int RED, int WT>
__device__ __forceinline__ void ring_fold4(const float x[][4], int W, float acc[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i] = x[0][i];
#pragma unroll
  for (int j = 1; j < Ranks<WT>::kMax; ++j)
    if (Ranks<WT>::has(j, W)) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        // reduce_apply(red, inbox, slot) (types.hpp:76-82): inbox = acc
        if (RED == COCONET_SUM) acc[i] = __fadd_rn(acc[i], x[j][i]);
        else if (RED == COCONET_MAX) acc[i] = acc[i] > x[j][i] ? acc[i] : x[j][i];
        else acc[i] = acc[i] < x[j][i] ? acc[i] : x[j][i];
      }
    }
}

// The same pull and fold with the quads kept packed until the fold (2
// registers per fp16 quad and rank instead of 4): the TMA kernels hold every
// rank's quads in flight while their stage fills.
template <typename G>
using GRaw = std::conditional_t<sizeof(G) == 4, float4, uint2>;

template <typename G, int WT>
__device__ __forceinline__ void ring_load_raw(char* const* base, int64_t off, int owner, int W, GRaw<G> x[]) {
#pragma unroll
  for (int j = 0; j < Ranks<WT>::kMax; ++j)
    if (Ranks<WT>::has(j, W)) x[j] = __ldg(reinterpret_cast<const GRaw<G>*>(base[rot<WT>(owner, j, W)] + off));
}

template <typename G, int WT>
__device__ __forceinline__ void ring_fold_raw(const GRaw<G> x[], int W, float acc[4]) {
#pragma unroll
  for (int j = 0; j < Ranks<WT>::kMax; ++j)
    if (Ranks<WT>::has(j, W)) {
      float y[4];
      if constexpr (sizeof(G) == 4) {
        y[0] = x[j].x; y[1] = x[j].y; y[2] = x[j].z; y[3] = x[j].w;
      } else {
        const G* h = reinterpret_cast<const G*>(&x[j]);
#pragma unroll
        for (int i = 0; i < 4; ++i) y[i] = to_f32(h[i]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = j == 0 ? y[i] : __fadd_rn(acc[i], y[i]);  // as ring_fold4
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

// Segment descriptor with its tensor's two heap offsets resolved.
struct SegD {
  int64_t toff, sidx, aoff, boff;
  int len, owner, tensor;
};

// Iterates this warp's descriptors [s, se) with stride `st` (D = Seg, or Item
// for the STREAMED schedule), prefetching the descriptor two ahead and the
// tensor offsets one ahead:
//   for (DescIter<Seg> it(...); it.valid(); it.next()) { SegD d = it.get(); ... }
// (no lambdas: capturing kernel parameters by reference spills them).
template <typename D>
struct DescIter {
  const D* segs;
  const int64_t* offs;
  int n;
  int64_t s, se, st;
  D d1, d2, d3;
  int64_t a1, b1, a2, b2;

  __device__ __forceinline__ DescIter(const D* segs_, const int64_t* offs_, int n_, int64_t s_, int64_t se_,
                                      int64_t st_)
      : segs(segs_), offs(offs_), n(n_), s(s_), se(se_), st(st_) {
    if (s < se) {
      d1 = segs[s];
      d2 = s + st < se ? segs[s + st] : d1;
      a1 = offs[meta_tensor(d1.meta)];
      b1 = offs[n + meta_tensor(d1.meta)];
      prefetch();
    }
  }
  __device__ __forceinline__ void prefetch() {
    d3 = s + 2 * st < se ? segs[s + 2 * st] : d2;
    a2 = offs[meta_tensor(d2.meta)];
    b2 = offs[n + meta_tensor(d2.meta)];
  }
  __device__ __forceinline__ bool valid() const { return s < se; }
  __device__ __forceinline__ int64_t index() const { return s; }
  __device__ __forceinline__ const D& raw() const { return d1; }
  __device__ __forceinline__ bool has_next() const { return s + st < se; }
  __device__ __forceinline__ const D& peek() const { return d2; }  // next descriptor (valid if has_next)
  __device__ __forceinline__ SegD get() const {
    return SegD{d1.toff, d1.sidx, a1, b1, meta_len(d1.meta), meta_owner(d1.meta), meta_tensor(d1.meta)};
  }
  __device__ __forceinline__ void next() {
    s += st;
    d1 = d2;
    d2 = d3;
    a1 = a2;
    b1 = b2;
    if (s < se) prefetch();
  }
};
using SegIter = DescIter<Seg>;

__device__ __forceinline__ void quad_range(const SegD& d, int64_t e0, int& lo, int& hi) {
  lo = int(max(int64_t(0), d.toff - e0));
  hi = int(min(int64_t(4), d.toff + d.len - e0));
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

// Quads [qs, qe) of one segment through Adam: U quads per lane in flight,
// clamped unconditional loads, then the ring fold, the element update and the
// stores (own m, v; p to every rank, or the own copy for ONE_SHOT).
template <typename G, int MATH, bool ONE_SHOT, int WT, int U>
__device__ __forceinline__ void adam_quads(char* const* s_base, const SegD& d, int64_t qs, int64_t qe, float* m,
                                           float* v, const char* pme, int me, int W, int lane, const AdamK& k) {
  for (int64_t qb = qs + lane; qb < qe; qb += 32 * U) {
    float g[U][Ranks<WT>::kMax][4], mm[U][4], vv[U][4], pp[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      // clamped, unconditional loads: the compiler can batch all U of them
      const int64_t q = min(qb + 32 * u, qe - 1);
      const int64_t e0 = q << 2;
      const int64_t si = d.sidx + (e0 - d.toff);
      ring_load4<G, COCONET_SUM, WT>(s_base, d.aoff + e0 * int64_t(sizeof(G)), d.owner, W, g[u]);
      ld4(m + si, mm[u]);
      ld4(v + si, vv[u]);
      ld4(reinterpret_cast<const float*>(pme + d.boff) + e0, pp[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = qb + 32 * u;
      if (q < qe) {
        const int64_t e0 = q << 2;
        int lo, hi;
        quad_range(d, e0, lo, hi);
        const int64_t si = d.sidx + (e0 - d.toff);
        float gs[4];
        ring_fold4<COCONET_SUM, WT>(g[u], W, gs);
#pragma unroll
        for (int i = 0; i < 4; ++i) adam_elem<MATH>(gs[i], mm[u][i], vv[u][i], pp[u][i], k);
        st4m(m + si, mm[u], lo, hi);
        st4m(v + si, vv[u], lo, hi);
        if (ONE_SHOT) {
          st4m(reinterpret_cast<float*>(s_base[me] + d.boff) + e0, pp[u], lo, hi);
        } else {
#pragma unroll
          for (int j = 0; j < Ranks<WT>::kMax; ++j)  // AG push, own copy included
            if (Ranks<WT>::has(j, W)) st4m(reinterpret_cast<float*>(s_base[j] + d.boff) + e0, pp[u], lo, hi);
        }
      }
    }
  }
}

// a.parts > 1 (small lists): each segment is split into `parts` quad ranges
// so the resident grid has work for every warp (C1: 256 segments per rank
// would otherwise keep 32 of 74 CTAs per rank busy).
template <typename G, int MATH, bool ONE_SHOT, int WT, int U>
__global__ void __launch_bounds__(kThreads, 2) adam_kernel(OptArgs a, AdamK k) {
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int W = WT > 0 ? WT : rs.world;
  const int me = rs.rank();
  if (!edge_barrier(rs, 0)) return;  // peers' gradients are complete
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sb = ONE_SHOT ? a.os_begin : a.seg_begin[me];
  const int64_t se = ONE_SHOT ? a.os_end : a.seg_begin[me + 1];
  float* m = reinterpret_cast<float*>(s_base[me] + a.m_off);
  float* v = reinterpret_cast<float*>(s_base[me] + a.v_off);
  const char* pme = s_base[me];
  const int64_t wid = int64_t(blockIdx.x) * kWarps + warp, wstride = int64_t(gridDim.x) * kWarps;
  if (a.parts > 1) {
    const int P = a.parts;
    for (int64_t it = wid; it < (se - sb) * P; it += wstride) {
      const Seg sg = a.segs[sb + it / P];
      const int part = int(it % P);
      const int tens = meta_tensor(sg.meta);
      const SegD d{sg.toff, sg.sidx, a.offs[tens], a.offs[a.n_tensors + tens], meta_len(sg.meta), meta_owner(sg.meta),
                   tens};
      const int64_t q0 = d.toff >> 2, nq = ((d.toff + d.len + 3) >> 2) - q0;
      adam_quads<G, MATH, ONE_SHOT, WT, U>(s_base, d, q0 + nq * part / P, q0 + nq * (part + 1) / P, m, v, pme, me,
                                           W, lane, k);
    }
  } else {
    for (SegIter it(a.segs, a.offs, a.n_tensors, sb + wid, se, wstride); it.valid(); it.next()) {
      const SegD d = it.get();
      adam_quads<G, MATH, ONE_SHOT, WT, U>(s_base, d, d.toff >> 2, (d.toff + d.len + 3) >> 2, m, v, pme, me, W,
                                           lane, k);
    }
  }
  edge_barrier(rs, 1);  // peers done reading our g and writing our p
}

// ---- NVLS (COCONET_ALGO_NVLS): the two-shot schedule through the multicast
// view of the world group's heaps (rs.mc, heap_cumem.cu). The reduce-scatter
// pull of W peers' quads becomes ONE multimem.ld_reduce (the NVSwitch sums
// the W copies and returns the total), and the all-gather push to W peers ONE
// multimem.st (the switch writes every copy). Per GPU per direction that is
// (W+1)/W*N*bytes on NVLink against 2(W-1)/W*N for the P2P two-shot. Quads
// cut by a segment edge are pushed rank by rank (no 16-bit scalar multimem
// store). The switch's summation order is its own: results are within fp32
// rounding of TWO_SHOT (16-bit g: the sum is returned rounded to the element
// type). fence.proxy.alias orders the multicast accesses against the unicast
// ones of the same memory at both barriers.
template <typename G>
__device__ __forceinline__ void mc_ld_reduce4(const char* addr, float o[4]) {
  if constexpr (sizeof(G) == 4) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3])
                 : "l"(addr)
                 : "memory");
  } else {
    uint32_t r[2];
    if constexpr (std::is_same<G, __half>::value)
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v2.f16x2 {%0,%1}, [%2];"
                   : "=r"(r[0]), "=r"(r[1])
                   : "l"(addr)
                   : "memory");
    else
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v2.bf16x2 {%0,%1}, [%2];"
                   : "=r"(r[0]), "=r"(r[1])
                   : "l"(addr)
                   : "memory");
    const G* h = reinterpret_cast<const G*>(r);
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = to_f32(h[i]);
  }
}

// Whole quad to every rank through the multicast address; a partial quad
// (lo > 0 or hi < 4) rank by rank through the unicast peer mappings.
template <typename T>
__device__ __forceinline__ void mc_st4(char* mc, char* const* base, int W, int64_t off, const float v[4], int lo,
                                       int hi) {
  if (lo == 0 && hi == 4) {
    if constexpr (sizeof(T) == 4) {
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + off), "f"(v[0]),
                   "f"(v[1]), "f"(v[2]), "f"(v[3])
                   : "memory");
    } else {
      T h[4] = {from_f32<T>(v[0]), from_f32<T>(v[1]), from_f32<T>(v[2]), from_f32<T>(v[3])};
      const uint2 u = *reinterpret_cast<const uint2*>(h);
      asm volatile("multimem.st.relaxed.sys.global.v2.f32 [%0], {%1,%2};" ::"l"(mc + off), "r"(u.x), "r"(u.y)
                   : "memory");
    }
  } else {
    for (int j = 0; j < W; ++j) st4m(reinterpret_cast<T*>(base[j] + off), v, lo, hi);
  }
}

__device__ __forceinline__ void fence_proxy_alias() { asm volatile("fence.proxy.alias;" ::: "memory"); }

template <typename G, int MATH>
__device__ __forceinline__ void adam_quads_nvls(char* const* s_base, char* mc, const SegD& d, int64_t qs,
                                                int64_t qe, float* m, float* v, const char* pme, int W, int lane,
                                                const AdamK& k) {
  constexpr int U = 2;
  for (int64_t qb = qs + lane; qb < qe; qb += 32 * U) {
    float g[U][4], mm[U][4], vv[U][4], pp[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = min(qb + 32 * u, qe - 1);
      const int64_t e0 = q << 2;
      const int64_t si = d.sidx + (e0 - d.toff);
      mc_ld_reduce4<G>(mc + d.aoff + e0 * int64_t(sizeof(G)), g[u]);
      ld4(m + si, mm[u]);
      ld4(v + si, vv[u]);
      ld4(reinterpret_cast<const float*>(pme + d.boff) + e0, pp[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = qb + 32 * u;
      if (q < qe) {
        const int64_t e0 = q << 2;
        int lo, hi;
        quad_range(d, e0, lo, hi);
        const int64_t si = d.sidx + (e0 - d.toff);
#pragma unroll
        for (int i = 0; i < 4; ++i) adam_elem<MATH>(g[u][i], mm[u][i], vv[u][i], pp[u][i], k);
        st4m(m + si, mm[u], lo, hi);
        st4m(v + si, vv[u], lo, hi);
        mc_st4<float>(mc, s_base, W, d.boff + e0 * 4, pp[u], lo, hi);
      }
    }
  }
}

template <typename G, int MATH>
__global__ void __launch_bounds__(kThreads, 2) adam_nvls_kernel(OptArgs a, AdamK k) {
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int W = rs.world, me = rs.rank();
  if (!edge_barrier(rs, 0)) return;  // peers' gradients are complete
  fence_proxy_alias();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sb = a.seg_begin[me], se = a.seg_begin[me + 1];
  float* m = reinterpret_cast<float*>(s_base[me] + a.m_off);
  float* v = reinterpret_cast<float*>(s_base[me] + a.v_off);
  const int64_t wid = int64_t(blockIdx.x) * kWarps + warp, wstride = int64_t(gridDim.x) * kWarps;
  const int P = a.parts;
  for (int64_t it = wid; it < (se - sb) * P; it += wstride) {
    const Seg sg = a.segs[sb + it / P];
    const int part = int(it % P);
    const int tens = meta_tensor(sg.meta);
    const SegD d{sg.toff, sg.sidx, a.offs[tens], a.offs[a.n_tensors + tens], meta_len(sg.meta), meta_owner(sg.meta),
                 tens};
    const int64_t q0 = d.toff >> 2, nq = ((d.toff + d.len + 3) >> 2) - q0;
    adam_quads_nvls<G, MATH>(s_base, rs.mc, d, q0 + nq * part / P, q0 + nq * (part + 1) / P, m, v, s_base[me], W,
                             lane, k);
  }
  fence_proxy_alias();
  edge_barrier(rs, 1);  // peers done reading our g and writing our p
}

// Tensor-list AllReduce (SUM) through the switch: rank r reduces its own
// chunk with multimem.ld_reduce and stores the total into every rank's out.
template <typename T>
__global__ void __launch_bounds__(kThreads, 2) allreduce_nvls_kernel(OptArgs a) {
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int W = rs.world, me = rs.rank();
  if (!edge_barrier(rs, 0)) return;
  fence_proxy_alias();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (SegIter it(a.segs, a.offs, a.n_tensors, a.seg_begin[me] + int64_t(blockIdx.x) * kWarps + warp,
                  a.seg_begin[me + 1], int64_t(gridDim.x) * kWarps);
       it.valid(); it.next()) {
    const SegD d = it.get();
    const int64_t q0 = d.toff >> 2, q1 = (d.toff + d.len + 3) >> 2;
    for (int64_t q = q0 + lane; q < q1; q += 32) {
      const int64_t e0 = q << 2;
      float acc[4];
      mc_ld_reduce4<T>(rs.mc + d.aoff + e0 * int64_t(sizeof(T)), acc);
      int lo, hi;
      quad_range(d, e0, lo, hi);
      mc_st4<T>(rs.mc, s_base, W, d.boff + e0 * int64_t(sizeof(T)), acc, lo, hi);
    }
  }
  fence_proxy_alias();
  edge_barrier(rs, 1);
}

// Tensor-list AllReduce (x -> out). TWO_SHOT = pull-RS of the own chunk +
// push-AG; ONE_SHOT = pull everything, write own copy (out != x).
template <typename T, int RED, bool ONE_SHOT, int WT, int U>
__global__ void __launch_bounds__(kThreads, 2) allreduce_kernel(OptArgs a) {
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int W = WT > 0 ? WT : rs.world;
  const int me = rs.rank();
  if (!edge_barrier(rs, 0)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sb = ONE_SHOT ? a.os_begin : a.seg_begin[me];
  const int64_t se = ONE_SHOT ? a.os_end : a.seg_begin[me + 1];
  for (SegIter it(a.segs, a.offs, a.n_tensors, sb + int64_t(blockIdx.x) * kWarps + warp, se,
                  int64_t(gridDim.x) * kWarps);
       it.valid(); it.next()) {
         const SegD d = it.get();
         const int64_t q0 = d.toff >> 2, q1 = (d.toff + d.len + 3) >> 2;
         for (int64_t qb = q0 + lane; qb < q1; qb += 32 * U) {
           float x[U][Ranks<WT>::kMax][4];
#pragma unroll
           for (int u = 0; u < U; ++u) {
             const int64_t q = min(qb + 32 * u, q1 - 1);  // clamped, unconditional loads
             ring_load4<T, RED, WT>(s_base, d.aoff + (q << 2) * int64_t(sizeof(T)), d.owner, W, x[u]);
           }
#pragma unroll
           for (int u = 0; u < U; ++u) {
             const int64_t q = qb + 32 * u;
             if (q < q1) {
               const int64_t e0 = q << 2;
               int lo, hi;
               quad_range(d, e0, lo, hi);
               float acc[4];
               ring_fold4<RED, WT>(x[u], W, acc);
               if (ONE_SHOT) {
                 st4m(reinterpret_cast<T*>(s_base[me] + d.boff) + e0, acc, lo, hi);
               } else {
#pragma unroll
                 for (int j = 0; j < Ranks<WT>::kMax; ++j)
                   if (Ranks<WT>::has(j, W)) st4m(reinterpret_cast<T*>(s_base[j] + d.boff) + e0, acc, lo, hi);
               }
             }
           }
         }
       }
  edge_barrier(rs, 1);
}

__device__ __forceinline__ float warp_sumf(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
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

// Per-tensor trust ratio of the golden: lr*sqrt(sum p^2)/sqrt(sum u^2)
// (expr text of tests/golden/lamb_fused_program.json, left-associative). The
// raw formula freezes a zero-norm tensor (ratio 0) and turns 0/0 into NaN;
// with k.guard (the torch-facing FusedLAMB) a zero norm gives ratio = lr, the
// apex / NVLAMB convention.
__device__ __forceinline__ double trust_ratio(double P, double U, const LambK& k) {
  if (k.guard && (P == 0.0 || U == 0.0)) return k.lr;
  return __ddiv_rn(__dmul_rn(k.lr, __dsqrt_rn(P)), __dsqrt_rn(U));
}

// LAMB, two passes inside one cooperative kernel:
//  pass 1: RS pull -> m, v update -> per-segment partial sums of p^2 and u^2
//  grid sync -> per-tensor partials of this rank (fixed segment order, so
//  deterministic) -> pushed into every peer's exchange area -> flag barrier
//  -> totals combined in rank order (state.hpp:163-167)
//  pass 2: trust ratio -> p update -> AG push.
// NV (COCONET_LAMB_NVLS, WT = 0): the RS pull is one multimem.ld_reduce per
// quad and the AG push one multimem.st through the multicast view (rs.mc);
// the per-tensor partials still go rank by rank (2 doubles per tensor).
template <typename G, int WT, int U, bool NV = false>
__global__ void __launch_bounds__(kThreads, 2) lamb_kernel(OptArgs a, LambK k) {
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int W = WT > 0 ? WT : rs.world;
  const int me = rs.rank();
  // No early return before the grid syncs: a CTA whose barrier timed out
  // skips its work but still arrives, so the grid cannot deadlock.
  const bool ok = edge_barrier(rs, 0);
  if constexpr (NV) fence_proxy_alias();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sb = a.seg_begin[me], se = ok ? a.seg_begin[me + 1] : sb;
  float* m = reinterpret_cast<float*>(s_base[me] + a.m_off);
  float* v = reinterpret_cast<float*>(s_base[me] + a.v_off);
  const char* pme = s_base[me];
  const int64_t wstride = int64_t(gridDim.x) * kWarps;
  const int64_t wid = int64_t(blockIdx.x) * kWarps + warp;
  // ---- pass 1
  for (SegIter it(a.segs, a.offs, a.n_tensors, sb + wid, se, wstride); it.valid(); it.next()) {
    const SegD d = it.get();
    const int64_t s = it.index();
    const int64_t q0 = d.toff >> 2, q1 = (d.toff + d.len + 3) >> 2;
    float sp = 0.f, su = 0.f;  // <=1024 squares per segment: fp32 is ample
    for (int64_t qb = q0 + lane; qb < q1; qb += 32 * U) {
      float g[U][NV ? 1 : Ranks<WT>::kMax][4], mm[U][4], vv[U][4], pp[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = min(qb + 32 * u, q1 - 1);  // clamped, unconditional loads
        {
          const int64_t e0 = q << 2;
          const int64_t si = d.sidx + (e0 - d.toff);
          if constexpr (NV) mc_ld_reduce4<G>(rs.mc + d.aoff + e0 * int64_t(sizeof(G)), g[u][0]);
          else ring_load4<G, COCONET_SUM, WT>(s_base, d.aoff + e0 * int64_t(sizeof(G)), me, W, g[u]);
          ld4(m + si, mm[u]);
          ld4(v + si, vv[u]);
          ld4(reinterpret_cast<const float*>(pme + d.boff) + e0, pp[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = qb + 32 * u;
        if (q < q1) {
          const int64_t e0 = q << 2;
          int lo, hi;
          quad_range(d, e0, lo, hi);
          const int64_t si = d.sidx + (e0 - d.toff);
          float gs[4];
          if constexpr (NV) {
#pragma unroll
            for (int i = 0; i < 4; ++i) gs[i] = g[u][0][i];
          } else {
            ring_fold4<COCONET_SUM, WT>(g[u], W, gs);
          }
          float fp = 0.f, fu = 0.f;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float mn = fmaf(k.fcm, gs[i], mm[u][i] * k.fb1);
            const float vn = fmaf(k.fcv * gs[i], gs[i], vv[u][i] * k.fb2);
            mm[u][i] = mn;
            vv[u][i] = vn;
            if (i >= lo && i < hi) {
              const float uu = lamb_u(mn, vn, pp[u][i], k);
              fp = fmaf(pp[u][i], pp[u][i], fp);
              fu = fmaf(uu, uu, fu);
            }
          }
          sp += fp;
          su += fu;
          st4m(m + si, mm[u], lo, hi);
          st4m(v + si, vv[u], lo, hi);
        }
      }
    }
    sp = warp_sumf(sp);
    su = warp_sumf(su);
    if (lane == 0) {
      k.seg_part[2 * s] = double(sp);
      k.seg_part[2 * s + 1] = double(su);
    }
  }
  __threadfence();
  cg::this_grid().sync();
  // ---- per-tensor partials of this rank -> every peer's exchange slot [me][t]
  const int64_t xch_off = int64_t(group_area(rs.group));
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
  for (SegIter it(a.segs, a.offs, a.n_tensors, sb + wid, se, wstride); it.valid(); it.next()) {
    const SegD d = it.get();
    double P = 0.0, Uu = 0.0;
#pragma unroll
    for (int q = 0; q < Ranks<WT>::kMax; ++q)  // rank order 0..W-1
      if (Ranks<WT>::has(q, W)) {
        P += __ldcg(xch_me + (int64_t(q) * a.n_tensors + d.tensor) * 2);
        Uu += __ldcg(xch_me + (int64_t(q) * a.n_tensors + d.tensor) * 2 + 1);
      }
    const float ratio = float(trust_ratio(P, Uu, k));
    const int64_t poff = d.boff;
    const int64_t q0 = d.toff >> 2, q1 = (d.toff + d.len + 3) >> 2;
    for (int64_t qb = q0 + lane; qb < q1; qb += 32 * U) {
      float mm[U][4], vv[U][4], pp[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = min(qb + 32 * u, q1 - 1);  // clamped, unconditional loads
        {
          const int64_t e0 = q << 2;
          const int64_t si = d.sidx + (e0 - d.toff);
          ld4(m + si, mm[u]);
          ld4(v + si, vv[u]);
          ld4(reinterpret_cast<const float*>(pme + poff) + e0, pp[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = qb + 32 * u;
        if (q < q1) {
          const int64_t e0 = q << 2;
          int lo, hi;
          quad_range(d, e0, lo, hi);
          float pn[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) pn[i] = pp[u][i] - ratio * lamb_u(mm[u][i], vv[u][i], pp[u][i], k);
          if constexpr (NV) {
            mc_st4<float>(rs.mc, s_base, W, poff + e0 * 4, pn, lo, hi);
          } else {
#pragma unroll
            for (int j = 0; j < Ranks<WT>::kMax; ++j)
              if (Ranks<WT>::has(j, W)) st4m(reinterpret_cast<float*>(s_base[j] + poff) + e0, pn, lo, hi);
          }
        }
      }
    }
  }
  if constexpr (NV) fence_proxy_alias();
  edge_barrier(rs, 1);
}

// LAMB element in EXACT math: eval_expr's double arithmetic on the golden's
// expression (tests/golden/lamb_fused_program.json; parser association,
// json_io.hpp:166-183, explicit _rn so nothing contracts):
//   m' = m*b1 + c1*g ; v' = v*b2 + (c2*g)*g
//   u  = (m'/bc1) / (sqrt(v'/bc2) + eps) + wd*p
__device__ __forceinline__ double lamb_u_exact(float g, float m, float v, float p, const LambK& k, double& mn,
                                               double& vn) {
  const double gd = g;
  mn = __dadd_rn(__dmul_rn(double(m), k.b1), __dmul_rn(k.c1, gd));
  vn = __dadd_rn(__dmul_rn(double(v), k.b2), __dmul_rn(__dmul_rn(k.c2, gd), gd));
  const double den = __dadd_rn(__dsqrt_rn(__ddiv_rn(vn, k.bc2)), k.eps);
  return __dadd_rn(__ddiv_rn(__ddiv_rn(mn, k.bc1), den), __dmul_rn(k.wd, double(p)));
}

// Between the two LAMB passes: this rank's per-tensor (P, U) partials, summed
// over its segments in CSR (fixed) order, into every rank's exchange slot
// [me][t] (state.hpp:163-167 combines them in rank order afterwards).
__device__ __forceinline__ void lamb_push_partials(const OptArgs& a, const LambK& k, char* const* s_base, int me,
                                                   int W, bool ok, int64_t wid, int64_t wstride, int lane) {
  const int64_t xch_off = int64_t(group_area(a.rs.group));
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
}

// LAMB in EXACT math (COCONET_MATH_EXACT): the reference evaluates the
// ReduceTensor pre-pass and the element pass from the SAME old m, v
// (state.hpp:139-190: the pre-pass does no Update stores, the element pass
// recomputes update(m, ...) from the old values). So pass 1 here is read-only
// (ring-order g, m, v, p -> u in double -> per-segment double sums of p*p and
// u*u) and pass 2 recomputes m', v', u from the same inputs, stores float(m'),
// float(v') and pushes float(p - ratio*u) (40 B/element at fp16 g against
// FAST's 38). Only the order of the two norm sums differs from the Engine's
// sequential accumulation.
template <typename G, int WT>
__global__ void __launch_bounds__(kThreads, 2) lamb_exact_kernel(OptArgs a, LambK k) {
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int W = WT > 0 ? WT : rs.world;
  const int me = rs.rank();
  const bool ok = edge_barrier(rs, 0);  // no early return before the grid syncs
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sb = a.seg_begin[me], se = ok ? a.seg_begin[me + 1] : sb;
  float* m = reinterpret_cast<float*>(s_base[me] + a.m_off);
  float* v = reinterpret_cast<float*>(s_base[me] + a.v_off);
  const char* pme = s_base[me];
  const int64_t wstride = int64_t(gridDim.x) * kWarps;
  const int64_t wid = int64_t(blockIdx.x) * kWarps + warp;
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      __threadfence();
      cg::this_grid().sync();
      lamb_push_partials(a, k, s_base, me, W, ok, wid, wstride, lane);
      __threadfence_system();
      cg::this_grid().sync();
      if (!rank_barrier(rs, 2)) return;
    }
    const double* xch_me = reinterpret_cast<const double*>(s_base[me] + group_area(rs.group));
    for (SegIter it(a.segs, a.offs, a.n_tensors, sb + wid, se, wstride); it.valid(); it.next()) {
      const SegD d = it.get();
      const int64_t s = it.index();
      double ratio = 0.0;
      if (pass == 1) {
        double P = 0.0, U = 0.0;
#pragma unroll
        for (int q = 0; q < Ranks<WT>::kMax; ++q)  // rank order 0..W-1
          if (Ranks<WT>::has(q, W)) {
            P += __ldcg(xch_me + (int64_t(q) * a.n_tensors + d.tensor) * 2);
            U += __ldcg(xch_me + (int64_t(q) * a.n_tensors + d.tensor) * 2 + 1);
          }
        ratio = trust_ratio(P, U, k);
      }
      const int64_t q0 = d.toff >> 2, q1 = (d.toff + d.len + 3) >> 2;
      double sp = 0.0, su = 0.0;
      for (int64_t q = q0 + lane; q < q1; q += 32) {
        float g[Ranks<WT>::kMax][4], mm[4], vv[4], pp[4];
        const int64_t e0 = q << 2;
        const int64_t si = d.sidx + (e0 - d.toff);
        ring_load4<G, COCONET_SUM, WT>(s_base, d.aoff + e0 * int64_t(sizeof(G)), me, W, g);
        ld4(m + si, mm);
        ld4(v + si, vv);
        ld4(reinterpret_cast<const float*>(pme + d.boff) + e0, pp);
        int lo, hi;
        quad_range(d, e0, lo, hi);
        float gs[4];
        ring_fold4<COCONET_SUM, WT>(g, W, gs);
        float pn[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          double mn, vn;
          const double u = lamb_u_exact(gs[i], mm[i], vv[i], pp[i], k, mn, vn);
          if (pass == 0) {
            if (i >= lo && i < hi) {
              sp = __dadd_rn(sp, __dmul_rn(double(pp[i]), double(pp[i])));
              su = __dadd_rn(su, __dmul_rn(u, u));
            }
          } else {
            mm[i] = float(mn);
            vv[i] = float(vn);
            pn[i] = float(__dsub_rn(double(pp[i]), __dmul_rn(ratio, u)));
          }
        }
        if (pass == 1) {
          st4m(m + si, mm, lo, hi);
          st4m(v + si, vv, lo, hi);
#pragma unroll
          for (int j = 0; j < Ranks<WT>::kMax; ++j)  // AllGather push
            if (Ranks<WT>::has(j, W)) st4m(reinterpret_cast<float*>(s_base[j] + d.boff) + e0, pn, lo, hi);
        }
      }
      if (pass == 0) {
        sp = warp_sum(sp);
        su = warp_sum(su);
        if (lane == 0) {
          k.seg_part[2 * s] = sp;
          k.seg_part[2 * s + 1] = su;
        }
      }
    }
  }
  edge_barrier(rs, 1);
}

// ---- LAMB, TMA schedule (W = 1): the GRID algorithm with its two streaming
// passes fed by the TMA engine. One persistent CTA per SM: warp 8 (one
// elected lane) walks the CTA's segments and issues cp.async.bulk copies of
// each 1024-element chunk of g, m, v, p into a ring of shared-memory stages
// (mbarrier complete_tx); warps 0-7 consume a chunk per stage, one quad per
// thread... (QPT quads per thread), write m, v (pass 1) or p (pass 2)
// straight to global memory and release the stage. Tens of KB per SM stay in flight without spending
// registers, which is what bounds the LDG kernel at 25% occupancy.
// Per-segment norm partials are summed in a fixed order (deterministic, not
// bit-identical to GRID's lane order); the per-tensor totals, the grid-wide
// syncs and the exchange are GRID's.
// NW consumer warps, QPT quads per consumer thread per chunk.
template <typename G, int NW, int QPT>
struct TmaStage {
  static constexpr int THREADS = (NW + 1) * 32;
  static constexpr int CHUNK_Q = NW * 32 * QPT;                                      // quads per chunk
  static constexpr int G_BYTES = (CHUNK_Q * 4 * int(sizeof(G)) + 16 + 15) / 16 * 16;  // + alignment slack
  static constexpr int A_BYTES = CHUNK_Q * 16;                                       // m, v, p
  static constexpr int BYTES = G_BYTES + 3 * A_BYTES;
};

struct TmaArgs {
  int stages;
};

// 32 segment descriptors of a CTA's list loaded at once by a warp (lane i:
// segment base + i*stride) and handed out with shuffles, so the
// descriptor -> tensor-offset chain costs one latency per 32 segments.
struct SegBatch {
  int64_t toff, sidx, aoff, boff;
  int len, tensor;
  __device__ __forceinline__ void load(const OptArgs& a, int64_t s, int64_t se) {
    if (s < se) {
      const Seg sg = a.segs[s];
      toff = sg.toff;
      sidx = sg.sidx;
      len = meta_len(sg.meta);
      tensor = meta_tensor(sg.meta);
      aoff = a.offs[tensor];
      boff = a.offs[a.n_tensors + tensor];
    } else {
      toff = sidx = aoff = boff = 0;
      len = 0;
      tensor = 0;
    }
  }
  __device__ __forceinline__ SegD get(int j, int me) const {
    const unsigned f = 0xffffffffu;
    return SegD{__shfl_sync(f, toff, j), __shfl_sync(f, sidx, j), __shfl_sync(f, aoff, j), __shfl_sync(f, boff, j),
                __shfl_sync(f, len, j), me, __shfl_sync(f, tensor, j)};
  }
};

// The producer warp of a TMA-ring kernel: walks the CTA's segments
// (batched descriptors) and, per chunk of ST::CHUNK_Q quads, waits for a free
// stage and issues the bulk copies of g (when with_g), m, v and p into it.
// Lane 0 issues; the warp returns the ring position it reached.
template <typename G, int NW, int QPT>
__device__ __forceinline__ void tma_produce(const OptArgs& a, char* const* s_base, int me, int64_t sb, int64_t se,
                                            uint8_t* stage0, uint64_t* full, uint64_t* empty, int S, bool with_g,
                                            int lane, uint32_t& st, uint32_t& ph) {
  using ST = TmaStage<G, NW, QPT>;
  const float* m = reinterpret_cast<const float*>(s_base[me] + a.m_off);
  const float* v = reinterpret_cast<const float*>(s_base[me] + a.v_off);
  const char* pme = s_base[me];
  const int64_t st32 = int64_t(gridDim.x) * 32;
  for (int64_t s0 = sb + blockIdx.x; s0 < se; s0 += st32) {
    SegBatch batch;
    batch.load(a, s0 + int64_t(lane) * gridDim.x, se);
    for (int j = 0; j < 32; ++j) {
      if (s0 + int64_t(j) * gridDim.x >= se) break;
      const SegD d = batch.get(j, me);
      if (lane != 0) continue;
      const int64_t q0 = d.toff >> 2, q1 = (d.toff + d.len + 3) >> 2;
      for (int64_t qa = q0; qa < q1; qa += ST::CHUNK_Q) {
        const int64_t qb = min(qa + int64_t(ST::CHUNK_Q), q1);
        mbar_wait(&empty[st], ph ^ 1u);
        uint8_t* dst = stage0 + size_t(st) * ST::BYTES;
        const uint32_t abytes = uint32_t(qb - qa) * 16u;
        const char* ga = pme + d.aoff + qa * 4 * int64_t(sizeof(G));
        const char* g0 = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(ga) & ~uintptr_t(15));
        const char* g1 = reinterpret_cast<const char*>(
            (reinterpret_cast<uintptr_t>(pme + d.aoff + qb * 4 * int64_t(sizeof(G))) + 15) & ~uintptr_t(15));
        const uint32_t gbytes = with_g ? uint32_t(g1 - g0) : 0u;
        const int64_t si = d.sidx + (qa * 4 - d.toff);
        mbar_expect_tx(&full[st], gbytes + 3u * abytes);
        if (with_g) bulk_load(dst, g0, gbytes, &full[st]);
        bulk_load(dst + ST::G_BYTES, m + si, abytes, &full[st]);
        bulk_load(dst + ST::G_BYTES + ST::A_BYTES, v + si, abytes, &full[st]);
        bulk_load(dst + ST::G_BYTES + 2 * ST::A_BYTES, pme + d.boff + qa * 16, abytes, &full[st]);
        if (++st == uint32_t(S)) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
  }
  __syncwarp();
  st = __shfl_sync(0xffffffffu, st, 0);
  ph = __shfl_sync(0xffffffffu, ph, 0);
}

template <typename G, int NW, int QPT, int WT>
__global__ void __launch_bounds__((NW + 1) * 32, 2) lamb_tma_kernel(OptArgs a, LambK k, TmaArgs ta) {
  using ST = TmaStage<G, NW, QPT>;
  constexpr int kTmaConsumerWarps = NW;
  constexpr int kTmaThreads = ST::THREADS;
  constexpr int kTmaChunkQ = ST::CHUNK_Q;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ char* s_base[kMaxRanks];
  __shared__ float s_red[2][NW][2];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int S = ta.stages;
  uint8_t* stage0 = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(stage0 + size_t(S) * ST::BYTES);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kTmaConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  const int me = rs.rank();
  const int W = WT > 0 ? WT : rs.world;
  const bool ok = edge_barrier(rs, 0);  // also publishes the barrier inits to the CTA
  const int64_t sb = a.seg_begin[me], se = ok ? a.seg_begin[me + 1] : sb;
  float* m = reinterpret_cast<float*>(s_base[me] + a.m_off);
  float* v = reinterpret_cast<float*>(s_base[me] + a.v_off);
  char* pme = s_base[me];
  const bool producer = warp == kTmaConsumerWarps;
  const int ctid = threadIdx.x;  // consumer thread 0..255
  uint32_t st = 0, ph = 0;       // ring slot and phase of the next chunk (both roles advance identically)
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      // ---- between the passes: per-tensor partials -> exchange -> totals (GRID)
      // Pass 1 wrote m, v with generic stores; pass 2's producer reads them
      // with cp.async.bulk (the async proxy): order the two proxies first.
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __threadfence();
      cg::this_grid().sync();
      const int64_t xch_off = int64_t(group_area(rs.group));
      const int64_t wstride = int64_t(gridDim.x) * (kTmaThreads / 32);
      const int64_t wid = int64_t(blockIdx.x) * (kTmaThreads / 32) + warp;
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
        if (lane < W) {  // this rank's partials into every rank's slot [me][t]
          double* xq = reinterpret_cast<double*>(s_base[lane] + xch_off);
          xq[(int64_t(me) * a.n_tensors + t) * 2] = sp;
          xq[(int64_t(me) * a.n_tensors + t) * 2 + 1] = su;
        }
      }
      __threadfence_system();
      cg::this_grid().sync();
      if (!rank_barrier(rs, 2)) return;  // every rank's partials have landed (no-op at W = 1)
    }
    const double* xch_me = reinterpret_cast<const double*>(s_base[me] + group_area(rs.group));
    if (producer) {
      // g comes through the ring only at W = 1; across ranks the consumers
      // pull it (peer memory is never a bulk-copy source)
      tma_produce<G, NW, QPT>(a, s_base, me, sb, se, stage0, full, empty, S, pass == 0 && W == 1, lane, st, ph);
    } else {
      int red = 0;  // s_red buffer of the next segment reduction
      const int64_t st32 = int64_t(gridDim.x) * 32;
      for (int64_t s0 = sb + blockIdx.x; s0 < se; s0 += st32) {
       SegBatch batch;
       batch.load(a, s0 + int64_t(lane) * gridDim.x, se);
       for (int j = 0; j < 32; ++j) {
        const int64_t s = s0 + int64_t(j) * gridDim.x;
        if (s >= se) break;
        const SegD d = batch.get(j, me);
        const int tens = d.tensor;
        const int64_t aoff = d.aoff, boff = d.boff;
        const int64_t q0 = d.toff >> 2, q1 = (d.toff + d.len + 3) >> 2;
        float ratio = 0.f;
        if (pass == 1) {
          double P = 0.0, U = 0.0;
#pragma unroll
          for (int q = 0; q < Ranks<WT>::kMax; ++q)  // rank order 0..W-1
            if (Ranks<WT>::has(q, W)) {
              P += __ldcg(xch_me + (int64_t(q) * a.n_tensors + tens) * 2);
              U += __ldcg(xch_me + (int64_t(q) * a.n_tensors + tens) * 2 + 1);
            }
          ratio = float(trust_ratio(P, U, k));
        }
        float sp = 0.f, su = 0.f;
        for (int64_t qa = q0; qa < q1; qa += kTmaChunkQ) {
          const int64_t qb = min(qa + int64_t(kTmaChunkQ), q1);
          // W > 1: this thread's g quads from every rank, in flight while
          // the stage fills (clamped, unconditional loads)
          GRaw<G> gw[QPT][Ranks<WT>::kMax];
          if (WT != 1 && pass == 0) {
#pragma unroll
            for (int qq = 0; qq < QPT; ++qq) {
              const int64_t q = min(qa + ctid + qq * (NW * 32), qb - 1);
              ring_load_raw<G, WT>(s_base, aoff + (q << 2) * int64_t(sizeof(G)), me, W, gw[qq]);
            }
          }
          mbar_wait(&full[st], ph);
          const uint8_t* src = stage0 + size_t(st) * ST::BYTES;
#pragma unroll
          for (int qq = 0; qq < QPT; ++qq) {
          const int64_t q = qa + ctid + qq * (NW * 32);
          if (q < qb) {
            const int64_t e0 = q << 2;
            int lo, hi;
            quad_range(d, e0, lo, hi);
            const int64_t si = d.sidx + (e0 - d.toff);
            const float4 mq = *reinterpret_cast<const float4*>(src + ST::G_BYTES + (q - qa) * 16);
            const float4 vq = *reinterpret_cast<const float4*>(src + ST::G_BYTES + ST::A_BYTES + (q - qa) * 16);
            const float4 pq = *reinterpret_cast<const float4*>(src + ST::G_BYTES + 2 * ST::A_BYTES + (q - qa) * 16);
            float mm[4] = {mq.x, mq.y, mq.z, mq.w}, vv[4] = {vq.x, vq.y, vq.z, vq.w}, pp[4] = {pq.x, pq.y, pq.z, pq.w};
            if (pass == 0) {
              const uintptr_t ga = reinterpret_cast<uintptr_t>(s_base[me] + aoff + qa * 4 * int64_t(sizeof(G)));
              const uintptr_t goff = (ga & 15u) + uintptr_t(q - qa) * 4u * sizeof(G);
              float gs[4];
              if (WT != 1) {  // ring order: rank me+1 first (runtime.hpp:302-305)
                ring_fold_raw<G, WT>(gw[qq], W, gs);
              } else if constexpr (sizeof(G) == 4) {
                const float4 gq = *reinterpret_cast<const float4*>(src + goff);
                gs[0] = gq.x; gs[1] = gq.y; gs[2] = gq.z; gs[3] = gq.w;
              } else {
                const uint2 gq = *reinterpret_cast<const uint2*>(src + goff);
                const G* h = reinterpret_cast<const G*>(&gq);
#pragma unroll
                for (int i = 0; i < 4; ++i) gs[i] = to_f32(h[i]);
              }
              float fp = 0.f, fu = 0.f;
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float mn = fmaf(k.fcm, gs[i], mm[i] * k.fb1);
                const float vn = fmaf(k.fcv * gs[i], gs[i], vv[i] * k.fb2);
                mm[i] = mn;
                vv[i] = vn;
                if (i >= lo && i < hi) {
                  const float uu = lamb_u(mn, vn, pp[i], k);
                  fp = fmaf(pp[i], pp[i], fp);
                  fu = fmaf(uu, uu, fu);
                }
              }
              sp += fp;
              su += fu;
              st4m(m + si, mm, lo, hi);
              st4m(v + si, vv, lo, hi);
            } else {
              float pn[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) pn[i] = pp[i] - ratio * lamb_u(mm[i], vv[i], pp[i], k);
#pragma unroll
              for (int j = 0; j < Ranks<WT>::kMax; ++j)  // AllGather push
                if (Ranks<WT>::has(j, W)) st4m(reinterpret_cast<float*>(s_base[j] + boff) + e0, pn, lo, hi);
            }
          }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[st]);
          if (++st == uint32_t(S)) {
            st = 0;
            ph ^= 1u;
          }
        }
        if (pass == 0) {  // segment partial: fixed-order sum over the 256 consumer threads
          sp = warp_sumf(sp);
          su = warp_sumf(su);
          if (lane == 0) {
            s_red[red][warp][0] = sp;
            s_red[red][warp][1] = su;
          }
          asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
          if (ctid == 0) {
            float tp = 0.f, tu = 0.f;
#pragma unroll
            for (int w = 0; w < kTmaConsumerWarps; ++w) {
              tp += s_red[red][w][0];
              tu += s_red[red][w][1];
            }
            k.seg_part[2 * s] = double(tp);
            k.seg_part[2 * s + 1] = double(tu);
          }
          red ^= 1;
        }
       }
      }
    }
  }
  edge_barrier(rs, 1);
}

// ---- LAMB, WINDOWED TMA schedule (group size 1). GRID/TMA read m, v and p
// twice from HBM (38 B/element at fp16 g) because pass 2 of ANY tensor waits
// for pass 1 of EVERY tensor (one grid-wide sync). Here the tensors are cut
// into windows of consecutive tensors (tlist_window_plan) and the persistent
// grid runs the phases
//     P1(w0); then per window w: P1head(w+1), P2(w), P1tail(w+1)
// so a window's pass 2 re-reads its m, v, p right after its pass 1 (plus a
// short head of the next window that covers the synchronisation), while
// they can still be in the 126 MB L2 (compulsory traffic: 26 B/element).
// Work is handed out DYNAMICALLY in batches of 4 chunk items (an atomic
// ticket per window and pass), so every CTA finishes a window within about
// one batch of the others. The producer warp draws the tickets and passes
// each chunk's descriptor to the consumers through shared memory next to its
// TMA stage. The CTA that completes a window's pass 1 last sums the per-item
// norm partials (fixed item order: deterministic) into per-tensor trust
// ratios and releases ready[w]; P2(w) waits for it. Deadlock-free: ready[w]
// needs only P1(w) items, all handed out before any CTA first waits; all CTAs
// are co-resident (cooperative launch). Element math is the TMA kernel's, so
// m, v are bit-identical to it and p equal within rounding of the norm sums.
struct LambWin {
  const int64_t* items;  // segment | chunk << 40, window by window, tensor-major
  const int64_t* wi;     // [K+1] window k = items [wi[k], wi[k+1])
  const int64_t* titem;  // [n_tensors+1] items of tensor t
  const int* tfirst;     // [K+1] window k = tensors [tfirst[k], tfirst[k+1])
  unsigned long long* tick;  // [K][2] cumulative tickets (batches) of P1 / P2
  uint32_t* cnt;         // [K] cumulative pass-1 arrivals
  uint32_t* ready;       // [K] = call once the window's ratios are published
  float2* ipart;         // [n_items] per-item CTA norm partials (sum p^2, sum u^2)
  float* ratio;          // [n_tensors]
  int K;
  uint32_t call;         // calls since the plan (and grid size) was set, this one included
  int64_t head;          // items of window w+1 run before P2(w)
};

constexpr int kWinBatch = 4;  // chunk items per ticket

// Phase j of: P1(0); then per window w: P1head(w+1), P2(w), P1tail(w+1)
// (the last window: P2 only). part: 0 whole, 1 head, 2 tail. 3K - 1 phases.
__device__ __forceinline__ void win_phase(int j, int K, int& pass, int& w, int& part) {
  if (j == 0) {
    pass = 0;
    w = 0;
    part = 0;
    return;
  }
  const int i = j - 1;
  const int ww = i / 3, r = i - 3 * ww;
  if (ww == K - 1 || r == 1) {
    pass = 1;
    w = ww;
    part = 0;
  } else {
    pass = 0;
    w = ww + 1;
    part = r == 0 ? 1 : 2;
  }
}

// Spin (relaxed polls: no L1 invalidation per poll) until *p == want, then
// ONE acquire fence.
__device__ __forceinline__ void wait_equal(const uint32_t* p, uint32_t want, const RankSet& rs) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  if (v != want) {
    const unsigned long long t0 = globaltimer();
    do {
      __nanosleep(64);
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
      if (globaltimer() - t0 > rs.timeout_ns) {
        atomicCAS(rs.status, 0, COCONET_ERR_TIMEOUT);
        break;
      }
    } while (v != want);
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// The ONCHIP window protocol's poll: acquire loads (no trailing gpu-scope
// fence: a fence waits for this thread's outstanding stores, microseconds
// under a saturated HBM; profiles/r02_lamb_onchip_trace.json). The caller
// shares what it observed with bar.sync.
__device__ __forceinline__ void wait_equal_acq(const uint32_t* p, uint32_t want, const RankSet& rs) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  if (v == want) return;
  const unsigned long long t0 = globaltimer();
  for (int i = 1;; ++i) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    if (v == want) return;
    if ((i & 255) == 0 && globaltimer() - t0 > rs.timeout_ns) {
      atomicCAS(rs.status, 0, COCONET_ERR_TIMEOUT);
      return;
    }
  }
}

// Chunk descriptor handed from the producer to the consumers with its stage.
struct ChunkD {
  int64_t toff, sidx, aoff, boff, item;  // item < 0: end of this CTA's phase
  int len, tensor, chunk, pad_;
};

__device__ __forceinline__ ChunkD load_chunk(const OptArgs& a, const int64_t* items, int64_t item) {
  ChunkD d;
  const int64_t it = items[item];
  const Seg sg = a.segs[it & ((int64_t(1) << 40) - 1)];
  d.item = item;
  d.chunk = int(it >> 40);
  d.toff = sg.toff;
  d.sidx = sg.sidx;
  d.len = meta_len(sg.meta);
  d.tensor = meta_tensor(sg.meta);
  d.aoff = a.offs[d.tensor];
  d.boff = a.offs[a.n_tensors + d.tensor];
  d.pad_ = 0;
  return d;
}

template <typename G, int NW, int QPT>
__global__ void __launch_bounds__((NW + 1) * 32, 2) lamb_win_kernel(OptArgs a, LambK k, TmaArgs ta, LambWin lw) {
  using ST = TmaStage<G, NW, QPT>;
  constexpr int kChunkQ = ST::CHUNK_Q;
  constexpr int kMaxStages = 16;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ char* s_base[kMaxRanks];
  __shared__ float s_red[2][NW][2];
  __shared__ ChunkD s_desc[kMaxStages];
  __shared__ int s_last;
  __shared__ double s_blk[2][NW];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int S = ta.stages;
  uint8_t* stage0 = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(stage0 + size_t(S) * ST::BYTES);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  const int me = rs.rank();
  edge_barrier(rs, 0);  // publishes the barrier inits to the CTA (group size 1: no peer)
  float* m = reinterpret_cast<float*>(s_base[me] + a.m_off);
  float* v = reinterpret_cast<float*>(s_base[me] + a.v_off);
  char* pme = s_base[me];
  const bool producer = warp == NW;
  const int ctid = threadIdx.x;
  const unsigned long long NG = gridDim.x;
  uint32_t st = 0, ph = 0;
  int red = 0;
  long long pend = -1;  // producer: the head's overshooting ticket, kept for the tail
  for (int j = 0; j < 3 * lw.K - 1; ++j) {
    int pass, w, part;
    win_phase(j, lw.K, pass, w, part);
    const int64_t wb = lw.wi[w], n = lw.wi[w + 1] - wb;
    const long long nbat = (n + kWinBatch - 1) / kWinBatch;
    if (pass == 1 && lane == 0) wait_equal(&lw.ready[w], lw.call, rs);  // the window's ratios are out
    __syncwarp();
    if (producer) {
      if (lane == 0) {
        if (pass == 1) asm volatile("fence.proxy.async.global;" ::: "memory");  // other CTAs' m, v stores
        unsigned long long* tk = &lw.tick[2 * w + pass];
        const unsigned long long base = (unsigned long long)(lw.call - 1) * ((unsigned long long)nbat + NG);
        const long long lim = part == 1 ? min(nbat, (long long)(lw.head / kWinBatch)) : nbat;
        long long t;
        if (part == 2) {  // the head's overshoot, or its failing draw (-2) already happened
          t = pend >= 0 ? pend : nbat;
          pend = -1;
        } else {
          t = (long long)(atomicAdd(tk, 1ull) - base);
        }
        while (t < lim) {
          const long long nxt = (long long)(atomicAdd(tk, 1ull) - base);  // in flight while t's chunks go out
          for (int q = 0; q < kWinBatch; ++q) {
            const int64_t item = t * kWinBatch + q;
            if (item >= n) break;
            const ChunkD d = load_chunk(a, lw.items, wb + item);
            const int64_t qa = (d.toff >> 2) + int64_t(d.chunk) * kChunkQ;
            const int64_t qb = min(qa + int64_t(kChunkQ), (d.toff + d.len + 3) >> 2);
            mbar_wait(&empty[st], ph ^ 1u);
            s_desc[st] = d;
            uint8_t* dst = stage0 + size_t(st) * ST::BYTES;
            const uint32_t abytes = uint32_t(qb - qa) * 16u;
            const char* ga = pme + d.aoff + qa * 4 * int64_t(sizeof(G));
            const char* g0 = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(ga) & ~uintptr_t(15));
            const char* g1 = reinterpret_cast<const char*>(
                (reinterpret_cast<uintptr_t>(pme + d.aoff + qb * 4 * int64_t(sizeof(G))) + 15) & ~uintptr_t(15));
            const uint32_t gbytes = pass == 0 ? uint32_t(g1 - g0) : 0u;
            const int64_t si = d.sidx + (qa * 4 - d.toff);
            mbar_expect_tx(&full[st], gbytes + 3u * abytes);
            if (pass == 0) bulk_load(dst, g0, gbytes, &full[st]);
            bulk_load(dst + ST::G_BYTES, m + si, abytes, &full[st]);
            bulk_load(dst + ST::G_BYTES + ST::A_BYTES, v + si, abytes, &full[st]);
            bulk_load(dst + ST::G_BYTES + 2 * ST::A_BYTES, pme + d.boff + qa * 16, abytes, &full[st]);
            if (++st == uint32_t(S)) {
              st = 0;
              ph ^= 1u;
            }
          }
          t = nxt;
        }
        if (part == 1) pend = t < nbat ? t : -2;  // the head's overshoot belongs to the tail
        // end of this CTA's phase: an empty stage with an end marker
        mbar_wait(&empty[st], ph ^ 1u);
        s_desc[st].item = -1;
        mbar_arrive(&full[st]);
        if (++st == uint32_t(S)) {
          st = 0;
          ph ^= 1u;
        }
      }
      __syncwarp();
      st = __shfl_sync(0xffffffffu, st, 0);
      ph = __shfl_sync(0xffffffffu, ph, 0);
      continue;
    }
    // ---- consumers
    int ratio_t = -1;
    float ratio = 0.f;
    for (;;) {
      mbar_wait(&full[st], ph);
      const ChunkD d0 = s_desc[st];
      if (d0.item < 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (++st == uint32_t(S)) {
          st = 0;
          ph ^= 1u;
        }
        break;
      }
      const SegD d{d0.toff, d0.sidx, d0.aoff, d0.boff, d0.len, me, d0.tensor};
      if (pass == 1 && d0.tensor != ratio_t) {
        ratio = __ldcg(&lw.ratio[d0.tensor]);
        ratio_t = d0.tensor;
      }
      const int64_t qa = (d.toff >> 2) + int64_t(d0.chunk) * kChunkQ;
      const int64_t qb = min(qa + int64_t(kChunkQ), (d.toff + d.len + 3) >> 2);
      const uint8_t* src = stage0 + size_t(st) * ST::BYTES;
      float sp = 0.f, su = 0.f;
#pragma unroll
      for (int qq = 0; qq < QPT; ++qq) {
        const int64_t q = qa + ctid + qq * (NW * 32);
        if (q < qb) {
          const int64_t e0 = q << 2;
          int lo, hi;
          quad_range(d, e0, lo, hi);
          const int64_t si = d.sidx + (e0 - d.toff);
          const float4 mq = *reinterpret_cast<const float4*>(src + ST::G_BYTES + (q - qa) * 16);
          const float4 vq = *reinterpret_cast<const float4*>(src + ST::G_BYTES + ST::A_BYTES + (q - qa) * 16);
          const float4 pq = *reinterpret_cast<const float4*>(src + ST::G_BYTES + 2 * ST::A_BYTES + (q - qa) * 16);
          float mm[4] = {mq.x, mq.y, mq.z, mq.w}, vv[4] = {vq.x, vq.y, vq.z, vq.w},
                pp[4] = {pq.x, pq.y, pq.z, pq.w};
          if (pass == 0) {
            const uintptr_t ga = reinterpret_cast<uintptr_t>(pme + d.aoff + qa * 4 * int64_t(sizeof(G)));
            const uintptr_t goff = (ga & 15u) + uintptr_t(q - qa) * 4u * sizeof(G);
            float gs[4];
            if constexpr (sizeof(G) == 4) {
              const float4 gq = *reinterpret_cast<const float4*>(src + goff);
              gs[0] = gq.x; gs[1] = gq.y; gs[2] = gq.z; gs[3] = gq.w;
            } else {
              const uint2 gq = *reinterpret_cast<const uint2*>(src + goff);
              const G* h = reinterpret_cast<const G*>(&gq);
#pragma unroll
              for (int i = 0; i < 4; ++i) gs[i] = to_f32(h[i]);
            }
            float fp = 0.f, fu = 0.f;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float mn = fmaf(k.fcm, gs[i], mm[i] * k.fb1);
              const float vn = fmaf(k.fcv * gs[i], gs[i], vv[i] * k.fb2);
              mm[i] = mn;
              vv[i] = vn;
              if (i >= lo && i < hi) {
                const float uu = lamb_u(mn, vn, pp[i], k);
                fp = fmaf(pp[i], pp[i], fp);
                fu = fmaf(uu, uu, fu);
              }
            }
            sp += fp;
            su += fu;
            st4m(m + si, mm, lo, hi);
            st4m(v + si, vv, lo, hi);
          } else {
            float pn[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) pn[i] = pp[i] - ratio * lamb_u(mm[i], vv[i], pp[i], k);
            st4m(reinterpret_cast<float*>(pme + d.boff) + e0, pn, lo, hi);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == uint32_t(S)) {
        st = 0;
        ph ^= 1u;
      }
      if (pass == 0) {  // the item's norm partial, CTA-reduced in fixed order
        sp = warp_sumf(sp);
        su = warp_sumf(su);
        if (lane == 0) {
          s_red[red][warp][0] = sp;
          s_red[red][warp][1] = su;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
        if (ctid == 0) {
          float tp = 0.f, tu = 0.f;
#pragma unroll
          for (int ww = 0; ww < NW; ++ww) {
            tp += s_red[red][ww][0];
            tu += s_red[red][ww][1];
          }
          lw.ipart[d0.item] = make_float2(tp, tu);
        }
        red ^= 1;
      }
    }
    if (pass == 0 && part != 1) {  // this CTA is done with the window's pass 1
      asm volatile("fence.proxy.async.global;" ::: "memory");  // m, v stores before their bulk readers
      asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
      if (ctid == 0) {
        __threadfence();
        const uint32_t old = atomicAdd(&lw.cnt[w], 1u);
        const int last = old + 1u == lw.call * uint32_t(gridDim.x);
        if (last) __threadfence();
        s_last = last;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
      if (s_last) {
        // the window's per-tensor trust ratios from the per-item partials in
        // item order: big tensors with every consumer thread, small ones a warp each
        for (int t = lw.tfirst[w]; t < lw.tfirst[w + 1]; ++t) {
          const int64_t i0 = lw.titem[t], i1 = lw.titem[t + 1];
          if (i1 - i0 <= 64) continue;
          double P = 0.0, U = 0.0;
          for (int64_t i = i0 + ctid; i < i1; i += NW * 32) {
            const float2 pu = __ldcg(&lw.ipart[i]);
            P += double(pu.x);
            U += double(pu.y);
          }
          P = warp_sum(P);
          U = warp_sum(U);
          if (lane == 0) {
            s_blk[0][warp] = P;
            s_blk[1][warp] = U;
          }
          asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
          if (ctid == 0) {
            double tp = 0.0, tu = 0.0;
            for (int ww = 0; ww < NW; ++ww) {
              tp += s_blk[0][ww];
              tu += s_blk[1][ww];
            }
            lw.ratio[t] = float(trust_ratio(tp, tu, k));
          }
          asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
        }
        for (int t = lw.tfirst[w] + warp; t < lw.tfirst[w + 1]; t += NW) {
          const int64_t i0 = lw.titem[t], i1 = lw.titem[t + 1];
          if (i1 - i0 > 64) continue;
          double P = 0.0, U = 0.0;
          for (int64_t i = i0 + lane; i < i1; i += 32) {
            const float2 pu = __ldcg(&lw.ipart[i]);
            P += double(pu.x);
            U += double(pu.y);
          }
          P = warp_sum(P);
          U = warp_sum(U);
          if (lane == 0) lw.ratio[t] = float(trust_ratio(P, U, k));
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
        if (ctid == 0) {
          __threadfence();
          st_release_sys(&lw.ready[w], lw.call);
        }
      }
    }
  }
  edge_barrier(rs, 1);
}

// ---- LAMB, ONCHIP schedule (group size 1). TMA/GRID pay 38 B/element at
// fp16 g because pass 2 re-reads m', v' and p from HBM to recompute u. Here
// pass 1 keeps u ON CHIP: every CTA (one per SM) holds the u of its chunk
// items of the current window in TMEM (tcgen05.st/ld, 32 chunks of 16
// columns) and in shared-memory slots next to the TMA ring, so pass 2 of a
// held item reads p only: 30 B/element (g 2 + m, v, p 12 read, m, v 8
// written; p 4 read and 4 written). The plan (tlist_onchip_plan) cuts the
// tensor-ordered chunk items into windows of whole tensors small enough that
// CTA c (items i == c mod G) holds all of its share; a tensor too large for
// one window spills its items beyond `hold` per CTA, which take TMA's pass 2
// (m', v', p re-read).
// Per CTA the order is P1(0), then for each window k: the first `head` items
// of P1(k+1), then P2(k) and the rest of P1(k+1) alternating, so the wait for
// window k's norms is covered by pass-1 work and the ring always mixes heavy
// (22 B) and light (8 B) items. Held items take ring slots in order
// (live <= hold + head = cap). Norms, released per tensor: each CTA sums
// its items of a tensor (thread partials, then the warps in fixed order) and
// queues the CTA partial to its sync warp, which stores it to part[t][cta],
// counts the arrival on the tensor's counter and, once a tensor's arrivals
// are complete, reduces its partials in CTA order (deterministic) into a
// shared-memory ratio table; pass 2 of a tensor waits for its own ratio only.
// Counters are zeroed by the last CTA out (graph replay). m', v' are TMA's
// bit for bit; u is the same lamb_u of the same fp32 m', v', p; only the
// norm summation order differs.
struct LambOC {
  const OcItem* items;
  const int64_t* wi;     // [K+1]
  const int* tfirst;     // [K+1]
  const int64_t* titem;  // [n_tensors+1]
  double2* part;         // [n_tensors][G]
  uint32_t* cnt;         // [K] pass-1 arrivals per window, [K] CTAs out; zero between launches
  int K;
  int hold, cap, head, head2, tslots;
  int slot_off;  // byte offset of the shared-memory u slots from the ring base
  int nosync;    // profiling only (COCONET_LAMB_OC_NOSYNC=1): skip the window waits, results invalid
  // profiling only (COCONET_LAMB_OC_TRACE=<heap offset>): per (window, CTA)
  // globaltimer at [0] pass 1 finished, [1] pass-2 wait reached, [2] released
  unsigned long long* trace;
};

__device__ __forceinline__ int64_t oc_first(int64_t b, int c, int G) {
  int64_t r = (int64_t(c) - b) % G;
  if (r < 0) r += G;
  return b + r;
}
__device__ __forceinline__ int oc_count(int64_t b, int64_t e, int c, int G) {
  const int64_t f = oc_first(b, c, G);
  return f < e ? int((e - 1 - f) / G + 1) : 0;
}

// The per-window item order shared by the producer and the consumers:
// head P1 items, then P2 and P1 alternating. next() = 0 done, 1 P1 (j), 2 P2 (j).
struct OcSeq {
  int n1, n2, h, h2, j1, j2;
  __device__ __forceinline__ void start(int n2_, int n1_, int head, int head2) {
    n1 = n1_;
    n2 = n2_;
    h = min(head, n1);
    h2 = min(head2, n1 - h);
    j1 = j2 = 0;
  }
  // P1 item j1 (held) reuses the slot of P2 item j1 - h, so P2 runs at
  // least j1 - h + 1 items ahead of it; after the head this alternates
  __device__ __forceinline__ int next(int& j) {
    if (j1 < h + h2) {
      j = j1++;
      return 1;
    }
    if (j2 >= n2 && j1 >= n1) return 0;
    if (j2 < n2 && (j1 >= n1 || j2 < j1 - h + 1)) {
      j = j2++;
      return 2;
    }
    j = j1++;
    return 1;
  }
};

// Item j of a CTA's n items of a window keeps its u on chip unless it is past
// the hold or one of the head2 items after the head (run early as cover for
// the previous window's norm wait, without a slot: they take the spilled path)
__device__ __forceinline__ bool oc_held(int j, int n, int hold, int head, int head2) {
  const int h = min(head, n), h2 = min(head2, n - h);
  return j < hold && !(j >= h && j < h + h2);
}

// 32 items of one stream (P1 or P2) of this CTA, loaded by the producer warp
// at once (lane l: item first + l*G) and handed out with shuffles.
struct OcBatch {
  int64_t toff, sidx, qa, aoff, boff;
  int len, tensor;
  __device__ __forceinline__ void load(const OptArgs& a, const OcItem* items, int64_t first, int G, int cnt,
                                       int lane) {
    if (lane < cnt) {
      const OcItem it = items[first + int64_t(lane) * G];
      toff = it.toff;
      sidx = it.sidx;
      qa = it.qa;
      len = it.len;
      tensor = it.tensor;
      aoff = a.offs[tensor];
      boff = a.offs[a.n_tensors + tensor];
    } else {
      toff = sidx = qa = aoff = boff = 0;
      len = tensor = 0;
    }
  }
};

struct OcDesc {
  int64_t toff, sidx, qa, aoff, boff;
  int len, tensor;
};

// What the consumers need of an item, resolved by the producer: 48 bytes
// (three 16-byte shared loads).
struct OcStage {
  float* mp;    // m' of the chunk's first element (v' at mp + v_minus_m)
  float* pp;    // p of the chunk's first element
  int nq;       // quads in the chunk
  int off0;     // element offset of the chunk's first quad from the segment start (>= -3)
  int len;      // segment length
  int tensor;
  int goff;     // byte offset of the chunk's g inside the stage
  int pad_;
};
__device__ __forceinline__ OcDesc oc_get(const OcBatch& b, int j) {
  const unsigned f = 0xffffffffu;
  return OcDesc{__shfl_sync(f, b.toff, j), __shfl_sync(f, b.sidx, j), __shfl_sync(f, b.qa, j),
                __shfl_sync(f, b.aoff, j), __shfl_sync(f, b.boff, j), __shfl_sync(f, b.len, j),
                __shfl_sync(f, b.tensor, j)};
}

template <int N>
__device__ __forceinline__ void tm_st(uint32_t taddr, const float* u) {
  if constexpr (N == 8) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "r"(__float_as_uint(u[0])), "r"(__float_as_uint(u[1])), "r"(__float_as_uint(u[2])),
                 "r"(__float_as_uint(u[3])), "r"(__float_as_uint(u[4])), "r"(__float_as_uint(u[5])),
                 "r"(__float_as_uint(u[6])), "r"(__float_as_uint(u[7]))
                 : "memory");
  } else {
    static_assert(N == 4, "x4 or x8");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr),
                 "r"(__float_as_uint(u[0])), "r"(__float_as_uint(u[1])), "r"(__float_as_uint(u[2])),
                 "r"(__float_as_uint(u[3]))
                 : "memory");
  }
}
template <int N>
__device__ __forceinline__ void tm_ld(uint32_t taddr, float* u) {
  uint32_t r[8];
  if constexpr (N == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
  } else {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr)
                 : "memory");
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < N; ++i) u[i] = __uint_as_float(r[i]);
}

constexpr int kOcTmemCols = 512;

// mbarrier wait for the consumers of the ONCHIP ring: the watchdog clock is
// read once per 64 polls (try_wait already suspends in hardware).
__device__ __forceinline__ void mbar_wait_lazy(uint64_t* bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const unsigned long long t0 = globaltimer();
  for (int i = 1;; ++i) {
    if (mbar_try(bar, parity)) return;
    if ((i & 63) == 0 && globaltimer() - t0 > 10000000000ull) __trap();
  }
}

template <typename G, int NW, int QPT>
__global__ void __launch_bounds__((NW + 2) * 32, 1) lamb_onchip_kernel(OptArgs a, LambK k, TmaArgs ta, LambOC oc) {
  using ST = TmaStage<G, NW, QPT>;
  constexpr int kChunkQ = ST::CHUNK_Q;
  constexpr int kFpt = QPT * 4;               // u floats per consumer thread per chunk
  constexpr int kSlotCols = kFpt * (NW / 4);  // TMEM columns of one chunk slot (128 lanes)
  static_assert(NW % 4 == 0 && (kFpt == 4 || kFpt == 8), "TMEM slot layout");
  constexpr int kMaxStages = 8;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ char* s_base[kMaxRanks];
  __shared__ float s_red[2][NW][2];
  __shared__ __align__(16) OcStage s_desc[kMaxStages];
  __shared__ float s_ratio[3][kOcMaxTensors];  // window % 3
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t s_p1done[2];  // window parity: one phase per two windows
  // per-tensor release: the consumers hand every finished tensor's CTA
  // partial (P, U, tensor) to the sync warp through this queue; the sync warp
  // publishes it, counts the arrival and turns globally complete tensors into
  // ratios, announced per window as (window << 16) | ratios ready
  constexpr int kQN = 32;
  __shared__ __align__(16) float4 s_q[kQN];
  __shared__ volatile uint32_t s_qhead, s_qtail;
  __shared__ volatile int s_p1windows;  // windows whose pass 1 this CTA completed (monotonic)
  __shared__ volatile uint32_t s_ready[3];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int S = ta.stages;
  uint8_t* stage0 = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(stage0 + size_t(S) * ST::BYTES);
  uint64_t* empty = full + S;
  uint8_t* slots = stage0 + oc.slot_off;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    mbar_init(&s_p1done[0], NW);
    mbar_init(&s_p1done[1], NW);
    s_qhead = s_qtail = 0u;
    s_p1windows = 0;
    s_ready[0] = s_ready[1] = s_ready[2] = 0xffffffffu;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(kOcTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  const int me = rs.rank();
  edge_barrier(rs, 0);  // publishes the barrier inits and the TMEM address (group size 1: no peer)
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  float* m = reinterpret_cast<float*>(s_base[me] + a.m_off);
  float* v = reinterpret_cast<float*>(s_base[me] + a.v_off);
  const int64_t v_minus_m = (a.v_off - a.m_off) / 4;
  char* pme = s_base[me];
  const int NG = int(gridDim.x), cta = int(blockIdx.x);
  const int K = oc.K;
  uint32_t st = 0, ph = 0;
  if (warp == NW) {
    // ---------------- producer
    OcBatch b1, b2;
    for (int kk = -1; kk < K; ++kk) {
      const int64_t w2b = kk >= 0 ? oc.wi[kk] : 0, w2e = kk >= 0 ? oc.wi[kk + 1] : 0;
      const int64_t w1b = kk + 1 < K ? oc.wi[kk + 1] : 0, w1e = kk + 1 < K ? oc.wi[kk + 2] : 0;
      const int n2 = kk >= 0 ? oc_count(w2b, w2e, cta, NG) : 0;
      const int n1 = kk + 1 < K ? oc_count(w1b, w1e, cta, NG) : 0;
      const int64_t f2 = oc_first(w2b, cta, NG), f1 = oc_first(w1b, cta, NG);
      OcSeq seq;
      seq.start(n2, n1, oc.head, oc.head2);
      bool spill_ok = false;
      int j, kind;
      while ((kind = seq.next(j)) != 0) {
        const bool p1 = kind == 1;
        if ((j & 31) == 0) {
          if (p1) b1.load(a, oc.items, f1 + int64_t(j) * NG, NG, min(32, n1 - j), lane);
          else b2.load(a, oc.items, f2 + int64_t(j) * NG, NG, min(32, n2 - j), lane);
        }
        const OcDesc d = oc_get(p1 ? b1 : b2, j & 31);
        if (lane == 0) {
          const bool held = oc_held(j, p1 ? n1 : n2, oc.hold, oc.head, oc.head2);
          if (!p1 && !held && !spill_ok) {  // m', v' of this window stored (generic proxy) by our consumers
            // window kk+2 is not issued yet, so its barrier is at most one phase ahead
            mbar_wait(&s_p1done[kk & 1], uint32_t(kk >> 1) & 1u);
            asm volatile("fence.proxy.async.global;" ::: "memory");
            spill_ok = true;
          }
          const int64_t qa = d.qa;
          const int64_t qb = min(qa + int64_t(kChunkQ), (d.toff + d.len + 3) >> 2);
          mbar_wait(&empty[st], ph ^ 1u);
          uint8_t* dst = stage0 + size_t(st) * ST::BYTES;
          const uint32_t abytes = uint32_t(qb - qa) * 16u;
          const int64_t si = d.sidx + (qa * 4 - d.toff);
          const uintptr_t ga = reinterpret_cast<uintptr_t>(pme + d.aoff + qa * 4 * int64_t(sizeof(G)));
          OcStage sd;
          sd.mp = m + si;
          sd.pp = reinterpret_cast<float*>(pme + d.boff) + qa * 4;
          sd.nq = int(qb - qa);
          sd.off0 = int(qa * 4 - d.toff);
          sd.len = d.len;
          sd.tensor = d.tensor;
          sd.goff = int(ga & 15u);
          sd.pad_ = 0;
          s_desc[st] = sd;
          if (p1) {
            const char* g0 = reinterpret_cast<const char*>(ga & ~uintptr_t(15));
            const char* g1 = reinterpret_cast<const char*>(
                (reinterpret_cast<uintptr_t>(pme + d.aoff + qb * 4 * int64_t(sizeof(G))) + 15) & ~uintptr_t(15));
            const uint32_t gbytes = uint32_t(g1 - g0);
            mbar_expect_tx(&full[st], gbytes + 3u * abytes);
            bulk_load(dst, g0, gbytes, &full[st]);
            bulk_load(dst + ST::G_BYTES, m + si, abytes, &full[st]);
            bulk_load(dst + ST::G_BYTES + ST::A_BYTES, v + si, abytes, &full[st]);
          } else if (!held) {
            mbar_expect_tx(&full[st], 3u * abytes);
            bulk_load(dst + ST::G_BYTES, m + si, abytes, &full[st]);
            bulk_load(dst + ST::G_BYTES + ST::A_BYTES, v + si, abytes, &full[st]);
          } else {
            mbar_expect_tx(&full[st], abytes);
          }
          bulk_load(dst + ST::G_BYTES + 2 * ST::A_BYTES, sd.pp, abytes, &full[st]);
        }
        if (++st == uint32_t(S)) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
  } else if (warp == NW + 1) {
    // ---------------- sync warp: per-tensor release of the norms
    uint32_t qt = 0;
    int w = 0, tn = K > 0 ? oc.tfirst[0] : 0;
    unsigned long long t_last = globaltimer();
    while (w < K) {
      bool moved = false;
      // every decision is lane 0's, broadcast: the warp stays converged for the shuffles
      const uint32_t qh = __shfl_sync(0xffffffffu, s_qhead, 0);
      if (qh != qt) {  // publish this CTA's finished tensors (at most kQN = 32 entries: one per lane)
        moved = true;
        __threadfence_block();
        int te_ = -1;
        if (uint32_t(lane) < qh - qt) {
          const float4 e = s_q[(qt + uint32_t(lane)) % kQN];
          te_ = __float_as_int(e.z);
          oc.part[int64_t(te_) * NG + cta] = make_double2(double(e.x), double(e.y));
        }
        __threadfence();  // the partials before the arrivals (only this warp's own stores are pending)
        if (te_ >= 0) atomicAdd(&oc.cnt[K + 1 + te_], 1u);
        __syncwarp();
        qt = qh;
        if (lane == 0) s_qtail = qt;
      }
      // window w's ratios in tensor order. Buffer w % 3 is free once this
      // CTA finished pass 1 of window w - 1, which orders it after its pass 2
      // of window w - 3 (the last reader of that buffer). A monotonic count,
      // not the s_p1done parity: that barrier may already be a phase further.
      const int te = oc.tfirst[w + 1];
      if (tn >= te) {
        ++w;
        moved = true;
      } else if (__shfl_sync(0xffffffffu, int(w < 3 || s_p1windows >= w), 0)) {
        // lanes probe the next 32 tensors' arrival counters at once
        const int tp = tn + lane;
        bool done_l = false;
        if (tp < te) {
          const int nl = int(min(oc.titem[tp + 1] - oc.titem[tp], int64_t(NG)));
          uint32_t c;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(&oc.cnt[K + 1 + tp]) : "memory");
          done_l = c == uint32_t(nl);
        }
        const uint32_t mask = __ballot_sync(0xffffffffu, done_l);
        __syncwarp();  // orders the acquiring lanes' loads before every lane's partial reads
        const int nb = mask == 0xffffffffu ? 32 : __ffs(~mask) - 1;  // complete tensors in a row
        const int tb = oc.tfirst[w], buf = w % 3;
        for (int b = 0; b < nb; ++b, ++tn) {
          const int64_t i0 = oc.titem[tn];
          const int n = int(min(oc.titem[tn + 1] - i0, int64_t(NG)));
          const int c0 = int(i0 % NG);
          double P = 0.0, U = 0.0;
          for (int r = lane; r < n; r += 32) {
            const int cc = c0 + r >= NG ? c0 + r - NG : c0 + r;
            const double2 pu = __ldcg(&oc.part[int64_t(tn) * NG + cc]);
            P += pu.x;
            U += pu.y;
          }
          P = warp_sum(P);
          U = warp_sum(U);
          if (lane == 0) {
            s_ratio[buf][tn - tb] = float(trust_ratio(P, U, k));
            __threadfence_block();
            s_ready[buf] = (uint32_t(w) << 16) | uint32_t(tn - tb + 1);
            if (oc.trace && tn + 1 == te) oc.trace[(int64_t(w) * NG + cta) * 4 + 2] = globaltimer();
          }
          __syncwarp();
        }
        moved |= nb > 0;
      }
      if (moved) {
        t_last = globaltimer();
      } else {
        __nanosleep(32);
        if (globaltimer() - t_last > 10000000000ull) __trap();  // watchdog: a CTA never arrived
      }
    }
  } else {
    // ---------------- consumers
    const int ctid = threadIdx.x;
    // TMEM: warp w owns lanes 32*(w%4).. and columns (w/4)*kFpt.. of every kSlotCols-column chunk slot
    const uint32_t tbase = tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * kFpt);
    int base2 = 0;  // ring slot of window kk's first held item
    int red = 0;
    for (int kk = -1; kk < K; ++kk) {
      const int64_t w2b = kk >= 0 ? oc.wi[kk] : 0, w2e = kk >= 0 ? oc.wi[kk + 1] : 0;
      const int64_t w1b = kk + 1 < K ? oc.wi[kk + 1] : 0, w1e = kk + 1 < K ? oc.wi[kk + 2] : 0;
      const int n2 = kk >= 0 ? oc_count(w2b, w2e, cta, NG) : 0;
      const int n1 = kk + 1 < K ? oc_count(w1b, w1e, cta, NG) : 0;
      int base1 = base2 + min(n2, oc.hold);
      if (base1 >= oc.cap) base1 -= oc.cap;
      const int t2 = kk >= 0 ? oc.tfirst[kk] : 0;
      OcSeq seq;
      seq.start(n2, n1, oc.head, oc.head2);
      int cur_t = -1;  // P1 tensor whose thread partials are open
      float sp = 0.f, su = 0.f;
      // flush the open tensor's CTA partial: fixed-order sum of the NW warps
      auto flush = [&]() {
        const float wp = warp_sumf(sp), wu = warp_sumf(su);
        if (lane == 0) {
          s_red[red][warp][0] = wp;
          s_red[red][warp][1] = wu;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
        if (ctid == 0) {
          float tp = 0.f, tu = 0.f;
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            tp += s_red[red][w][0];
            tu += s_red[red][w][1];
          }
          const uint32_t h = s_qhead;
          while (h - s_qtail >= uint32_t(kQN)) __nanosleep(32);  // full: the sync warp drains it
          s_q[h % kQN] = make_float4(tp, tu, __int_as_float(cur_t), 0.f);
          __threadfence_block();
          s_qhead = h + 1;
        }
        red ^= 1;
        sp = su = 0.f;
      };
      // this CTA's pass 1 of window kk+1 is complete: partials out, m', v'
      // ordered before the spilled bulk re-reads, arrival counted
      auto finish_p1 = [&]() {
        if (cur_t >= 0) flush();
        cur_t = -1;
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_p1done[(kk + 1) & 1]);
        asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
        if (ctid == 0) s_p1windows = kk + 2;  // every consumer warp is past pass 1 of window kk + 1
      };
      if (kk + 1 < K && n1 == 0) finish_p1();
      int j, kind;
      while ((kind = seq.next(j)) != 0) {
        const bool p1 = kind == 1;
        mbar_wait_lazy(&full[st], ph);
        const OcStage d = s_desc[st];
        if (p1 && d.tensor != cur_t) {
          if (cur_t >= 0) flush();
          cur_t = d.tensor;
        }
        const bool held = oc_held(j, p1 ? n1 : n2, oc.hold, oc.head, oc.head2);
        int slot = (p1 ? base1 : base2) + j;
        if (slot >= oc.cap) slot -= oc.cap;
        const uint8_t* src = stage0 + size_t(st) * ST::BYTES;
        float u[kFpt];
        if (!p1 && held) {
          if (slot < oc.tslots) {
            tm_ld<kFpt>(tbase + uint32_t(slot * kSlotCols), u);
          } else {
            const uint8_t* sl = slots + size_t(slot - oc.tslots) * (kChunkQ * 16);
#pragma unroll
            for (int qq = 0; qq < QPT; ++qq) {
              const float4 x = *reinterpret_cast<const float4*>(sl + qq * (NW * 32 * 16) + ctid * 16);
              u[qq * 4 + 0] = x.x; u[qq * 4 + 1] = x.y; u[qq * 4 + 2] = x.z; u[qq * 4 + 3] = x.w;
            }
          }
        }
        float ratio = 0.f;
        if (!p1) {  // this tensor's ratio: published by the sync warp once every CTA's pass 1 of it is in
          const uint32_t want = uint32_t(d.tensor - t2);
          if (oc.nosync != 1) {
            uint32_t rv = s_ready[kk % 3];
            for (int i = 1; (rv >> 16) != uint32_t(kk) || (rv & 0xffffu) <= want; ++i) {
              __nanosleep(20);
              rv = s_ready[kk % 3];
              if ((i & 1023) == 0 && failed(rs)) break;
            }
            __threadfence_block();
          }
          ratio = s_ratio[kk % 3][want];
        }
        float fp = 0.f, fu = 0.f;
#pragma unroll
        for (int qq = 0; qq < QPT; ++qq) {
          const int qi = ctid + qq * (NW * 32);  // quad inside the chunk
          const bool in = qi < d.nq;
          const int er = 4 * qi + d.off0;  // its first element's offset in the segment
          const int lo = in ? max(0, -er) : 4, hi = min(4, d.len - er);
          const bool whole = lo == 0 && hi == 4;
          const float4 pq = *reinterpret_cast<const float4*>(src + ST::G_BYTES + 2 * ST::A_BYTES + qi * 16);
          const float pp[4] = {pq.x, pq.y, pq.z, pq.w};
          if (p1) {
            const float4 mq = *reinterpret_cast<const float4*>(src + ST::G_BYTES + qi * 16);
            const float4 vq = *reinterpret_cast<const float4*>(src + ST::G_BYTES + ST::A_BYTES + qi * 16);
            float mm[4] = {mq.x, mq.y, mq.z, mq.w}, vv[4] = {vq.x, vq.y, vq.z, vq.w};
            float gs[4];
            if constexpr (sizeof(G) == 4) {
              const float4 gq = *reinterpret_cast<const float4*>(src + d.goff + qi * 16);
              gs[0] = gq.x; gs[1] = gq.y; gs[2] = gq.z; gs[3] = gq.w;
            } else {
              const uint2 gq = *reinterpret_cast<const uint2*>(src + d.goff + qi * 8);
              const G* h = reinterpret_cast<const G*>(&gq);
#pragma unroll
              for (int i = 0; i < 4; ++i) gs[i] = to_f32(h[i]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float mn = fmaf(k.fcm, gs[i], mm[i] * k.fb1);
              const float vn = fmaf(k.fcv * gs[i], gs[i], vv[i] * k.fb2);
              mm[i] = mn;
              vv[i] = vn;
              const float uu = lamb_u(mn, vn, pp[i], k);
              u[qq * 4 + i] = uu;
              const bool ok = whole || (i >= lo && i < hi);  // (stage bytes past the chunk are garbage)
              fp = ok ? fmaf(pp[i], pp[i], fp) : fp;
              fu = ok ? fmaf(uu, uu, fu) : fu;
            }
            if (whole) {
              store4(d.mp + 4 * qi, mm);
              store4(d.mp + v_minus_m + 4 * qi, vv);
            } else if (in) {
              st4m(d.mp + 4 * qi, mm, lo, hi);
              st4m(d.mp + v_minus_m + 4 * qi, vv, lo, hi);
            }
          } else {
            if (!held) {
              const float4 mq = *reinterpret_cast<const float4*>(src + ST::G_BYTES + qi * 16);
              const float4 vq = *reinterpret_cast<const float4*>(src + ST::G_BYTES + ST::A_BYTES + qi * 16);
              const float mm[4] = {mq.x, mq.y, mq.z, mq.w}, vv[4] = {vq.x, vq.y, vq.z, vq.w};
#pragma unroll
              for (int i = 0; i < 4; ++i) u[qq * 4 + i] = lamb_u(mm[i], vv[i], pp[i], k);
            }
            float pn[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) pn[i] = pp[i] - ratio * u[qq * 4 + i];
            if (whole) store4(d.pp + 4 * qi, pn);
            else if (in) st4m(d.pp + 4 * qi, pn, lo, hi);
          }
        }
        if (p1 && held) {
          if (slot < oc.tslots) {
            tm_st<kFpt>(tbase + uint32_t(slot * kSlotCols), u);
          } else {
            uint8_t* sl = slots + size_t(slot - oc.tslots) * (kChunkQ * 16);
#pragma unroll
            for (int qq = 0; qq < QPT; ++qq)
              *reinterpret_cast<float4*>(sl + qq * (NW * 32 * 16) + ctid * 16) =
                  make_float4(u[qq * 4 + 0], u[qq * 4 + 1], u[qq * 4 + 2], u[qq * 4 + 3]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (++st == uint32_t(S)) {
          st = 0;
          ph ^= 1u;
        }
        if (p1) {
          sp += fp;
          su += fu;
          if (j == n1 - 1) finish_p1();
        }
      }
      base2 = base1;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  edge_barrier(rs, 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kOcTmemCols) : "memory");
  // every CTA has passed all of its window waits: the last one out zeroes the
  // counters for the next launch (so a captured graph replays correctly)
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&oc.cnt[K], 1u) == uint32_t(NG) - 1u) {
      for (int i = 0; i <= K + a.n_tensors; ++i) oc.cnt[i] = 0u;
      __threadfence();
    }
  }
}

// ---- Adam, TMA schedule (W = 1): one pass, the producer of lamb_tma_kernel
// streaming g, m, v, p into the shared-memory ring and NW consumer warps
// applying adam_elem (EXACT or FAST) and writing m, v, p.
template <typename G, int NW, int QPT, int MATH, int WT>
__global__ void __launch_bounds__((NW + 1) * 32, 2) adam_tma_kernel(OptArgs a, AdamK k, TmaArgs ta) {
  using ST = TmaStage<G, NW, QPT>;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ char* s_base[kMaxRanks];
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int S = ta.stages;
  uint8_t* stage0 = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(stage0 + size_t(S) * ST::BYTES);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  const int me = rs.rank();
  const int W = WT > 0 ? WT : rs.world;
  const bool ok = edge_barrier(rs, 0);
  const int64_t sb = a.seg_begin[me], se = ok ? a.seg_begin[me + 1] : sb;
  float* m = reinterpret_cast<float*>(s_base[me] + a.m_off);
  float* v = reinterpret_cast<float*>(s_base[me] + a.v_off);
  char* pme = s_base[me];
  uint32_t st = 0, ph = 0;
  if (warp == NW) {
    // across ranks g is pulled by the consumers (never a bulk copy from peer memory)
    tma_produce<G, NW, QPT>(a, s_base, me, sb, se, stage0, full, empty, S, W == 1, lane, st, ph);
  } else {
    const int ctid = threadIdx.x;
    const int64_t st32 = int64_t(gridDim.x) * 32;
    for (int64_t s0 = sb + blockIdx.x; s0 < se; s0 += st32) {
      SegBatch batch;
      batch.load(a, s0 + int64_t(lane) * gridDim.x, se);
      for (int j = 0; j < 32; ++j) {
        if (s0 + int64_t(j) * gridDim.x >= se) break;
        const SegD d = batch.get(j, me);
        const int64_t q0 = d.toff >> 2, q1 = (d.toff + d.len + 3) >> 2;
        for (int64_t qa = q0; qa < q1; qa += ST::CHUNK_Q) {
          const int64_t qb = min(qa + int64_t(ST::CHUNK_Q), q1);
          GRaw<G> gw[QPT][Ranks<WT>::kMax];  // W > 1: every rank's quads, in flight while the stage fills
          if (WT != 1) {
#pragma unroll
            for (int qq = 0; qq < QPT; ++qq) {
              const int64_t q = min(qa + ctid + qq * (NW * 32), qb - 1);
              ring_load_raw<G, WT>(s_base, d.aoff + (q << 2) * int64_t(sizeof(G)), me, W, gw[qq]);
            }
          }
          mbar_wait(&full[st], ph);
          const uint8_t* src = stage0 + size_t(st) * ST::BYTES;
          const uintptr_t ga = reinterpret_cast<uintptr_t>(pme + d.aoff + qa * 4 * int64_t(sizeof(G)));
#pragma unroll
          for (int qq = 0; qq < QPT; ++qq) {
            const int64_t q = qa + ctid + qq * (NW * 32);
            if (q < qb) {
              const int64_t e0 = q << 2;
              int lo, hi;
              quad_range(d, e0, lo, hi);
              const int64_t si = d.sidx + (e0 - d.toff);
              const float4 mq = *reinterpret_cast<const float4*>(src + ST::G_BYTES + (q - qa) * 16);
              const float4 vq = *reinterpret_cast<const float4*>(src + ST::G_BYTES + ST::A_BYTES + (q - qa) * 16);
              const float4 pq = *reinterpret_cast<const float4*>(src + ST::G_BYTES + 2 * ST::A_BYTES + (q - qa) * 16);
              float mm[4] = {mq.x, mq.y, mq.z, mq.w}, vv[4] = {vq.x, vq.y, vq.z, vq.w}, pp[4] = {pq.x, pq.y, pq.z, pq.w};
              const uintptr_t goff = (ga & 15u) + uintptr_t(q - qa) * 4u * sizeof(G);
              float gs[4];
              if (WT != 1) {
                ring_fold_raw<G, WT>(gw[qq], W, gs);
              } else if constexpr (sizeof(G) == 4) {
                const float4 gq = *reinterpret_cast<const float4*>(src + goff);
                gs[0] = gq.x; gs[1] = gq.y; gs[2] = gq.z; gs[3] = gq.w;
              } else {
                const uint2 gq = *reinterpret_cast<const uint2*>(src + goff);
                const G* h = reinterpret_cast<const G*>(&gq);
#pragma unroll
                for (int i = 0; i < 4; ++i) gs[i] = to_f32(h[i]);
              }
#pragma unroll
              for (int i = 0; i < 4; ++i) adam_elem<MATH>(gs[i], mm[i], vv[i], pp[i], k);
              st4m(m + si, mm, lo, hi);
              st4m(v + si, vv, lo, hi);
#pragma unroll
              for (int jr = 0; jr < Ranks<WT>::kMax; ++jr)  // AllGather push
                if (Ranks<WT>::has(jr, W)) st4m(reinterpret_cast<float*>(s_base[jr] + d.boff) + e0, pp, lo, hi);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[st]);
          if (++st == uint32_t(S)) {
            st = 0;
            ph ^= 1u;
          }
        }
      }
    }
  }
  edge_barrier(rs, 1);
}

// STREAMED-LAMB bookkeeping (tlist_stream_plan).
struct LambS {
  const Item* items;
  const int64_t* p1_first;  // [rank][tensor]
  const uint32_t* holders;  // [tensor] rank bitmask
  uint32_t* cnt;            // [rank][tensor] pass-1 completion counters
  double* part;             // [item] sum p^2, sum u^2 (pass-1 items)
  int64_t item_begin[kMaxRanks + 1];
  int64_t rdy_off;          // ready flags [src rank][tensor] in the group area
  uint32_t call;            // launches of this schedule so far, this one included
};

// Sum of n (p^2, u^2) pairs at part[2*first ...], lane-strided in list order
// then a butterfly: the same additions, in the same order, as the GRID
// kernel's CSR walk (the pass-1 items of a tensor are its CSR list), so both
// schedules produce bit-identical norms.
__device__ __forceinline__ void reduce_parts(const double* part, int64_t first, int64_t n, int lane,
                                             double& P, double& Uu) {
  P = 0.0;
  Uu = 0.0;
  int64_t i = lane;
  for (; i + 96 < n; i += 128) {  // four independent 16-byte loads in flight per lane
    double2 x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = __ldcg(reinterpret_cast<const double2*>(part + 2 * (first + i + 32 * j)));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      P += x[j].x;
      Uu += x[j].y;
    }
  }
  for (; i < n; i += 32) {
    const double2 x = __ldcg(reinterpret_cast<const double2*>(part + 2 * (first + i)));
    P += x.x;
    Uu += x.y;
  }
  P = warp_sum(P);
  Uu = warp_sum(Uu);
}

__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Per-CTA state of the STREAMED kernel that lives in shared memory.
struct StreamSmem {
  // speculative norms of upcoming pass-2 items, 3 slots by item parity mod 3
  // (a slot is rewritten two items after it was read; each item has a barrier)
  double2 spec[3][kMaxRanks];
  int rdy[3][kMaxRanks];
};

// Warp 0 of a STREAMED CTA: publish the pending pass-1 completion of tensor t
// (fence + per-tensor counter). Returns (warp-uniform) whether this CTA
// completed the tensor and must run stream_reduce for it.
__device__ __forceinline__ bool stream_count(uint32_t* cnt, uint32_t call, int64_t nseg, int t) {
  int last = 0;
  if ((threadIdx.x & 31) == 0) {
    fence_acq_rel_gpu();  // this CTA's m, v and partial (ordered by the barrier) before the count
    const uint32_t old = atomicAdd(cnt + t, 1u);
    last = old + 1u == call * uint32_t(nseg);
  }
  return __shfl_sync(0xffffffffu, last, 0) != 0;
}

// Warp 0 of the CTA that completed tensor t: reduce its pass-1 partials in
// list order and push them, with a ready flag, to every peer. Runs between
// items (no data registers live).
__device__ __noinline__ void stream_reduce(char* const* s_base, const double* part, int64_t first, int64_t nseg,
                                           int64_t xch_off, int64_t rdy_off, uint32_t epoch, int n, int W, int me,
                                           int t) {
  const int lane = threadIdx.x & 31;
  fence_acq_rel_gpu();
  double P, Uu;
  reduce_parts(part, first, nseg, lane, P, Uu);
  if (lane < W) {
    double* xq = reinterpret_cast<double*>(s_base[lane] + xch_off);
    *reinterpret_cast<double2*>(xq + (int64_t(me) * n + t) * 2) = make_double2(P, Uu);
    __threadfence_system();
    st_release_sys(reinterpret_cast<uint32_t*>(s_base[lane] + xch_off + rdy_off) + int64_t(me) * n + t, epoch);
  }
}

// Threads 32 + q (q < W, warp 1: warp 0 is busy publishing counts) of a
// STREAMED CTA: non-blocking readiness check and (P, U) partials of rank q
// for tensor t, into speculation slot `sl`.
__device__ __forceinline__ void stream_speculate(StreamSmem& ss, const LambS& ls, const uint32_t* rdy_me,
                                              const double* xch_me, uint32_t epoch, int n, int t, int sl) {
  const int q = threadIdx.x - 32;
  int r = 1;
  double2 x = make_double2(0.0, 0.0);
  if ((ls.holders[t] >> q) & 1u) {
    r = int32_t(ld_acquire_sys(rdy_me + int64_t(q) * n + t) - epoch) >= 0;
    if (r) x = __ldcg(reinterpret_cast<const double2*>(xch_me + (int64_t(q) * n + t) * 2));
  }
  ss.spec[sl][q] = x;
  ss.rdy[sl][q] = r;
}

// LAMB, STREAMED schedule (coconet_lamb_sched): one persistent cooperative
// grid walks the rank's item list (tlist_stream_plan's order), ONE CTA PER
// ITEM, so only gridDim.x items (~1.2M elements) are in flight at once and a
// pass-2 item is never dequeued before its tensor's pass 1 is done.
//  pass-1 item: RS pull -> m, v update -> per-quad (p^2, u^2) partials in smem,
//    summed by warp 0 in the GRID kernel's lane order (lane l: quads l+32j, j
//    ascending, then a butterfly), so the segment partial is bit-identical.
//    Its completion (fence + per-tensor counter) is published by warp 0 one
//    item LATER, after that item's loads are in flight; the CTA that
//    completes a tensor reduces its partials in list order and pushes them,
//    with a ready flag, to every peer;
//  pass-2 item: its tensor's ready flags and (P, U) partials were read
//    speculatively while the previous item's loads were in flight (a blocking
//    wait only if they were not ready yet); combined in rank order
//    (state.hpp:163-167) -> trust ratio -> p update -> AG push. Its m, v, p
//    were touched `lag` elements earlier, so the re-reads hit L2, not HBM.
template <typename G, int WT, int NT, int U>
__global__ void __launch_bounds__(NT, 512 / NT) lamb_stream_kernel(OptArgs a, LambK k, LambS ls) {
  constexpr int kChunkQuads = NT * U;  // quads per CTA sweep (NT * U = 256: 1024 elements)
  __shared__ char* s_base[kMaxRanks];
  __shared__ float2 s_part[kChunkQuads];
  __shared__ StreamSmem ss;
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  const int W = WT > 0 ? WT : rs.world;
  const int me = rs.rank();
  const bool ok = edge_barrier(rs, 0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n_tensors;
  const int64_t ib = ls.item_begin[me], ie = ok ? ls.item_begin[me + 1] : ib;
  float* m = reinterpret_cast<float*>(s_base[me] + a.m_off);
  float* v = reinterpret_cast<float*>(s_base[me] + a.v_off);
  const char* pme = s_base[me];
  const int64_t* ptr = k.csr_ptr + k.csr_begin[me];
  uint32_t* cnt = ls.cnt + int64_t(me) * n;
  const int64_t* p1_first = ls.p1_first + int64_t(me) * n;
  const int64_t xch_off = int64_t(group_area(rs.group));
  const double* xch_me = reinterpret_cast<const double*>(s_base[me] + xch_off);
  const uint32_t* rdy_me = reinterpret_cast<const uint32_t*>(s_base[me] + xch_off + ls.rdy_off);
  int pend_t = -1;  // warp 0: pass-1 item whose completion is not yet published
  int red_t = -1;   // warp 0: tensor this CTA completed, to reduce after the item
  int slot = 0;  // this item's speculation slot
  if (tid < W) ss.rdy[0][tid] = 0;  // the first item is never speculated
  static_assert(NT >= 64, "speculation runs on warp 1");
  for (DescIter<Item> it(ls.items, a.offs, n, ib + blockIdx.x, ie, gridDim.x); it.valid(); it.next()) {
    const SegD d = it.get();
    const int t = d.tensor;
    const int nslot = slot == 2 ? 0 : slot + 1;
    const bool spec_next = it.has_next() && meta_pass(it.peek().meta) == 1;
    const int64_t q0 = d.toff >> 2, q1 = (d.toff + d.len + 3) >> 2;
    if (meta_pass(it.raw().meta) == 0) {
      float sp = 0.f, su = 0.f;  // warp 0's lane accumulators (GRID order)
      for (int64_t qc = q0; qc < q1; qc += kChunkQuads) {
        float g[U][Ranks<WT>::kMax][4], mm[U][4], vv[U][4], pp[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t q = min(qc + tid + NT * u, q1 - 1);  // clamped, unconditional loads
          const int64_t e0 = q << 2;
          const int64_t si = d.sidx + (e0 - d.toff);
          ring_load4<G, COCONET_SUM, WT>(s_base, d.aoff + e0 * int64_t(sizeof(G)), me, W, g[u]);
          ld4(m + si, mm[u]);
          ld4(v + si, vv[u]);
          ld4(reinterpret_cast<const float*>(pme + d.boff) + e0, pp[u]);
        }
        if (qc == q0) {  // overlap the previous item's publish and the next item's speculation
          if (warp == 0 && pend_t >= 0) {
            if (stream_count(cnt, ls.call, ptr[pend_t + 1] - ptr[pend_t], pend_t)) red_t = pend_t;
            pend_t = -1;
          }
          if (spec_next && tid >= 32 && tid < 32 + W) stream_speculate(ss, ls, rdy_me, xch_me, rs.epoch, n, meta_tensor(it.peek().meta), nslot);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t q = qc + tid + NT * u;
          float fp = 0.f, fu = 0.f;
          if (q < q1) {
            const int64_t e0 = q << 2;
            int lo, hi;
            quad_range(d, e0, lo, hi);
            const int64_t si = d.sidx + (e0 - d.toff);
            float gs[4];
            ring_fold4<COCONET_SUM, WT>(g[u], W, gs);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float mn = fmaf(k.fcm, gs[i], mm[u][i] * k.fb1);
              const float vn = fmaf(k.fcv * gs[i], gs[i], vv[u][i] * k.fb2);
              mm[u][i] = mn;
              vv[u][i] = vn;
              if (i >= lo && i < hi) {
                const float uu = lamb_u(mn, vn, pp[u][i], k);
                fp = fmaf(pp[u][i], pp[u][i], fp);
                fu = fmaf(uu, uu, fu);
              }
            }
            st4m(m + si, mm[u], lo, hi);
            st4m(v + si, vv[u], lo, hi);
          }
          s_part[tid + NT * u] = make_float2(fp, fu);  // +0.0 past the end: no effect
        }
        __syncthreads();
        if (warp == 0) {
          const int nq = int(min(int64_t(kChunkQuads), q1 - qc));
          for (int j = lane; j < nq; j += 32) {
            const float2 x = s_part[j];
            sp += x.x;
            su += x.y;
          }
        }
        __syncthreads();
      }
      if (warp == 0) {
        sp = warp_sumf(sp);
        su = warp_sumf(su);
        if (lane == 0)
          *reinterpret_cast<double2*>(ls.part + 2 * it.index()) = make_double2(double(sp), double(su));
        pend_t = t;
      }
    } else {
      __syncthreads();  // this item's speculation slot is visible
      bool ready = true;
#pragma unroll
      for (int q = 0; q < Ranks<WT>::kMax; ++q)
        if (Ranks<WT>::has(q, W)) ready &= ss.rdy[slot][q] != 0;
      const double2* xs = ss.spec[slot];  // the rank partials: speculated, or filled below
      if (!ready) {  // rare: block on the flags BEFORE loading m, v (pass 1 may still be writing them)
        if (warp == 0 && pend_t >= 0) {  // we may hold the count it needs ...
          if (stream_count(cnt, ls.call, ptr[pend_t + 1] - ptr[pend_t], pend_t)) red_t = pend_t;
          pend_t = -1;
        }
        if (warp == 0 && red_t >= 0) {  // ... or the reduction
          stream_reduce(s_base, ls.part, p1_first[red_t], ptr[red_t + 1] - ptr[red_t], xch_off, ls.rdy_off,
                        rs.epoch, n, W, me, red_t);
          red_t = -1;
        }
        bool okw = true;
        if (tid < W && ((ls.holders[t] >> tid) & 1u)) okw = wait_flag(rdy_me + int64_t(tid) * n + t, rs.epoch, rs);
        if (tid < W)
          ss.spec[slot][tid] = ((ls.holders[t] >> tid) & 1u) && okw
                                   ? __ldcg(reinterpret_cast<const double2*>(xch_me + (int64_t(tid) * n + t) * 2))
                                   : make_double2(0.0, 0.0);
        if (!__syncthreads_and(okw)) break;  // watchdog fired: skip, never hang
      }
      for (int64_t qc = q0; qc < q1; qc += kChunkQuads) {
        float mm[U][4], vv[U][4], pp[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t q = min(qc + tid + NT * u, q1 - 1);
          const int64_t e0 = q << 2;
          const int64_t si = d.sidx + (e0 - d.toff);
          load4_cg(m + si, mm[u]);
          load4_cg(v + si, vv[u]);
          load4_cg(reinterpret_cast<const float*>(pme + d.boff) + e0, pp[u]);
        }
        if (qc == q0) {
          if (warp == 0 && pend_t >= 0) {
            if (stream_count(cnt, ls.call, ptr[pend_t + 1] - ptr[pend_t], pend_t)) red_t = pend_t;
            pend_t = -1;
          }
          if (spec_next && tid >= 32 && tid < 32 + W) stream_speculate(ss, ls, rdy_me, xch_me, rs.epoch, n, meta_tensor(it.peek().meta), nslot);
        }
        double P = 0.0, Uu = 0.0;
#pragma unroll
        for (int q = 0; q < Ranks<WT>::kMax; ++q)  // rank order 0..W-1; non-holders add +0.0
          if (Ranks<WT>::has(q, W)) {
            P += xs[q].x;
            Uu += xs[q].y;
          }
        const float ratio = float(trust_ratio(P, Uu, k));
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t q = qc + tid + NT * u;
          if (q < q1) {
            const int64_t e0 = q << 2;
            int lo, hi;
            quad_range(d, e0, lo, hi);
            float pn[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) pn[i] = pp[u][i] - ratio * lamb_u(mm[u][i], vv[u][i], pp[u][i], k);
#pragma unroll
            for (int j = 0; j < Ranks<WT>::kMax; ++j)
              if (Ranks<WT>::has(j, W)) st4m(reinterpret_cast<float*>(s_base[j] + d.boff) + e0, pn, lo, hi);
          }
        }
      }
    }
    if (warp == 0 && red_t >= 0) {
      stream_reduce(s_base, ls.part, p1_first[red_t], ptr[red_t + 1] - ptr[red_t], xch_off, ls.rdy_off, rs.epoch,
                    n, W, me, red_t);
      red_t = -1;
    }
    slot = nslot;
  }
  if (warp == 0 && pend_t >= 0) {
    if (stream_count(cnt, ls.call, ptr[pend_t + 1] - ptr[pend_t], pend_t))
      stream_reduce(s_base, ls.part, p1_first[pend_t], ptr[pend_t + 1] - ptr[pend_t], xch_off, ls.rdy_off,
                    rs.epoch, n, W, me, pend_t);
  }
  edge_barrier(rs, 1);
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
  a->parts = 1;
  return COCONET_OK;
}

int64_t max_rank_segs(const coconet_tlist* tl, int W, bool one_shot) {
  if (one_shot) return tl->os_end - tl->os_begin;
  int64_t mx = 0;
  for (int r = 0; r < W; ++r) mx = std::max(mx, tl->seg_begin[r + 1] - tl->seg_begin[r]);
  return mx;
}

int launch_opt(coconet_ctx* c, coconet_tlist* tl, const void* func, void** args, bool one_shot,
               cudaStream_t stream, int parts = 1) {
  int W = c->groups[size_t(tl->group)].size;
  int64_t want = (max_rank_segs(tl, W, one_shot) * parts + kWarps - 1) / kWarps;
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
  // AUTO: the crossover measured on B200 (profiles/r01_oneshot_twoshot_crossover.json):
  // up to 2^14 elements both variants sit on the launch + flag-barrier floor,
  // from 2^16 two-shot wins, so one-shot only for tiny lists (the paper's V100
  // crossover was 2^16); at W == 1 both are the same
  // local update.
  return W > 1 && tl->total <= (int64_t(1) << 12);
}

// ---- instantiation tables: group size specialised for 1, 2, 4, 8 ranks,
// generic (runtime W) otherwise; unroll depth by how many loads a quad needs.
template <int WT> constexpr int unroll_for() { return WT == 1 ? 4 : (WT == 2 ? 2 : (WT == 4 ? 2 : 1)); }

template <typename G, int MATH, bool OS, int WT>
const void* adam_fn() {
  constexpr int U = MATH == COCONET_MATH_EXACT ? (WT == 1 ? 2 : 1) : unroll_for<WT>();
  return reinterpret_cast<const void*>(&adam_kernel<G, MATH, OS, WT, U>);
}

template <typename G, int MATH, bool OS>
const void* adam_w(int W) {
  switch (W) {
    case 1: return adam_fn<G, MATH, OS, 1>();
    case 2: return adam_fn<G, MATH, OS, 2>();
    case 4: return adam_fn<G, MATH, OS, 4>();
    case 8: return adam_fn<G, MATH, OS, 8>();
    default: return adam_fn<G, MATH, OS, 0>();
  }
}

template <typename G>
const void* adam_pick(int math, bool os, int W) {
  if (math == COCONET_MATH_EXACT) return os ? adam_w<G, COCONET_MATH_EXACT, true>(W) : adam_w<G, COCONET_MATH_EXACT, false>(W);
  return os ? adam_w<G, COCONET_MATH_FAST, true>(W) : adam_w<G, COCONET_MATH_FAST, false>(W);
}

template <typename G>
const void* adam_nvls_pick(int math) {
  return math == COCONET_MATH_EXACT ? reinterpret_cast<const void*>(&adam_nvls_kernel<G, COCONET_MATH_EXACT>)
                                    : reinterpret_cast<const void*>(&adam_nvls_kernel<G, COCONET_MATH_FAST>);
}

template <typename T, int RED, bool OS>
const void* ar_w(int W) {
  switch (W) {
    // 16-bit elements move 8 bytes per quad: twice the quads in flight
    case 1: return reinterpret_cast<const void*>(&allreduce_kernel<T, RED, OS, 1, sizeof(T) == 2 ? 8 : 4>);
    case 2: return reinterpret_cast<const void*>(&allreduce_kernel<T, RED, OS, 2, 4>);
    case 4: return reinterpret_cast<const void*>(&allreduce_kernel<T, RED, OS, 4, 2>);
    case 8: return reinterpret_cast<const void*>(&allreduce_kernel<T, RED, OS, 8, 1>);
    default: return reinterpret_cast<const void*>(&allreduce_kernel<T, RED, OS, 0, 1>);
  }
}

template <typename T>
const void* ar_pick(int red, bool os, int W) {
  if (red == COCONET_MAX) return os ? ar_w<T, COCONET_MAX, true>(W) : ar_w<T, COCONET_MAX, false>(W);
  if (red == COCONET_MIN) return os ? ar_w<T, COCONET_MIN, true>(W) : ar_w<T, COCONET_MIN, false>(W);
  return os ? ar_w<T, COCONET_SUM, true>(W) : ar_w<T, COCONET_SUM, false>(W);
}

template <typename G>
const void* lamb_pick(int W) {
  switch (W) {
    case 1: return reinterpret_cast<const void*>(&lamb_kernel<G, 1, 4>);
    case 2: return reinterpret_cast<const void*>(&lamb_kernel<G, 2, 2>);
    case 4: return reinterpret_cast<const void*>(&lamb_kernel<G, 4, 2>);
    case 8: return reinterpret_cast<const void*>(&lamb_kernel<G, 8, 1>);
    default: return reinterpret_cast<const void*>(&lamb_kernel<G, 0, 1>);
  }
}

template <typename G>
const void* lamb_exact_pick(int W) {
  switch (W) {
    case 1: return reinterpret_cast<const void*>(&lamb_exact_kernel<G, 1>);
    case 2: return reinterpret_cast<const void*>(&lamb_exact_kernel<G, 2>);
    case 4: return reinterpret_cast<const void*>(&lamb_exact_kernel<G, 4>);
    case 8: return reinterpret_cast<const void*>(&lamb_exact_kernel<G, 8>);
    default: return reinterpret_cast<const void*>(&lamb_exact_kernel<G, 0>);
  }
}

template <typename G>
const void* lamb_stream_pick(int W) {
  switch (W) {
    case 1: return reinterpret_cast<const void*>(&lamb_stream_kernel<G, 1, 64, 4>);
    case 2: return reinterpret_cast<const void*>(&lamb_stream_kernel<G, 2, 128, 2>);
    case 4: return reinterpret_cast<const void*>(&lamb_stream_kernel<G, 4, 128, 2>);
    case 8: return reinterpret_cast<const void*>(&lamb_stream_kernel<G, 8, 256, 1>);
    default: return reinterpret_cast<const void*>(&lamb_stream_kernel<G, 0, 256, 1>);
  }
}

// Default STREAMED lag: 2^21 elements (m, v, p = 24 MB): covers the grid's
// in-flight window (2 CTAs x 148 SMs x 4096-element items = 1.2M elements)
// while tensor + lag stay inside the 126 MB L2 for tensors up to ~4M.
constexpr int64_t kDefaultLag = int64_t(1) << 21;

// The TMA ring pays off when a segment spans several 2048-element chunks: at
// 1024-element buckets its per-segment cost dominates (LAMB 4.1 ms vs GRID
// 2.4 ms), from 4096 up it wins (LAMB 2.06 vs 2.26 ms, Adam EXACT 2.0 vs
// 2.5 ms at 16384). Group size 1 only (peer bulk copies untested).
constexpr int64_t kTmaMinBucket = 4096;
// WINDOWED LAMB: elements per window (COCONET_LAMB_WIN_ELEMS or
// coconet_lamb_params.lag_elems override it)
constexpr int64_t kDefaultWindow = int64_t(2) << 20;
// ONCHIP LAMB in AUTO from this many elements per shard (group size 1)
constexpr int64_t kOnchipMinElems = int64_t(1) << 20;
constexpr int kOcHead2 = 1;  // spilled cover items per window (COCONET_LAMB_OC_HEAD2 overrides)

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
  const bool nvls = hp->algo == COCONET_ALGO_NVLS;
  if (nvls && (!c->mc_base || tl->group != 0))
    return set_error(COCONET_ERR_UNSUPPORTED, "COCONET_ALGO_NVLS needs coconet_nvls_setup on the world group "
                                              "(coconet_nvls_supported reports why it is unavailable)");
  const bool os = !nvls && resolve_one_shot(hp->algo, tl, W);
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
  // two-shot tables with large buckets: the TMA ring (local m, v, p and, at
  // W = 1, g; across ranks the consumers pull g and push p). COCONET_ADAM_TMA:
  // 0 keeps the LDG kernel, 1 forces the ring whatever the bucket size.
  const char* te = getenv("COCONET_ADAM_TMA");
  const bool tma = te ? te[0] == '1' : tl->bucket_cap >= (W == 1 ? kTmaMinBucket : 4 * kTmaMinBucket);
  if (!os && !nvls && tma) {
    const void* fn = nullptr;
    int sbytes = 0, threads = 0;
    auto pick = [&](auto tag_g) {
      using Gt = decltype(tag_g);
      using ST = TmaStage<Gt, 8, 2>;
      auto by_w = [&](auto math_tag) -> const void* {
        constexpr int M = decltype(math_tag)::value;
        return W == 1   ? reinterpret_cast<const void*>(&adam_tma_kernel<Gt, 8, 2, M, 1>)
               : W == 2 ? reinterpret_cast<const void*>(&adam_tma_kernel<Gt, 8, 2, M, 2>)
               : W == 4 ? reinterpret_cast<const void*>(&adam_tma_kernel<Gt, 8, 2, M, 4>)
               : W == 8 ? reinterpret_cast<const void*>(&adam_tma_kernel<Gt, 8, 2, M, 8>)
                        : reinterpret_cast<const void*>(&adam_tma_kernel<Gt, 8, 2, M, 0>);
      };
      fn = hp->math == COCONET_MATH_EXACT ? by_w(std::integral_constant<int, COCONET_MATH_EXACT>{})
                                          : by_w(std::integral_constant<int, COCONET_MATH_FAST>{});
      sbytes = ST::BYTES;
      threads = ST::THREADS;
    };
    if (g_elem == COCONET_F32) pick(float{});
    else if (g_elem == COCONET_F16) pick(__half{});
    else pick(__nv_bfloat16{});
    const char* ce = getenv("COCONET_ADAM_TMA_CTAS");  // ring sized as for this many CTAs per SM
    const int per_sm = ce ? std::max(1, std::min(4, atoi(ce))) : 3;
    TmaArgs ta;
    ta.stages = std::min(16, (200 << 10) / per_sm / sbytes);
    const size_t smem = size_t(ta.stages) * size_t(sbytes) + size_t(ta.stages) * 16 + 128;
    rc = ensure_smem(c, fn, smem);
    if (rc) return rc;
    const int lr = local_ranks(c, tl->group);
    int blocks = 0;
    rc = coop_blocks(c, fn, threads, smem, tl->group, int64_t(c->sm_count) * per_sm / lr, &blocks);
    if (rc) return rc;
    void* args[] = {&a, &k, &ta};
    return coop_launch(c, fn, dim3(unsigned(blocks), unsigned(lr)), dim3(unsigned(threads)), args, smem, stream);
  }
  const void* fn = nvls ? (g_elem == COCONET_F32   ? adam_nvls_pick<float>(hp->math)
                           : g_elem == COCONET_F16 ? adam_nvls_pick<__half>(hp->math)
                                                   : adam_nvls_pick<__nv_bfloat16>(hp->math))
                   : g_elem == COCONET_F32 ? adam_pick<float>(hp->math, os, W)
                   : g_elem == COCONET_F16 ? adam_pick<__half>(hp->math, os, W)
                                           : adam_pick<__nv_bfloat16>(hp->math, os, W);
  // split segments while the resident grid has idle warps (small lists)
  int per_sm = 0;
  rc = occupancy(c, fn, kThreads, 0, &per_sm);
  if (rc) return rc;
  const int64_t warps = int64_t(per_sm) * c->sm_count / local_ranks(c, tl->group) * kWarps;
  const int64_t segs = std::max<int64_t>(1, max_rank_segs(tl, W, os));
  a.parts = 1;
  while (a.parts < 8 && segs * a.parts * 2 <= warps) a.parts *= 2;
  void* args[] = {&a, &k};
  return launch_opt(c, tl, fn, args, os, stream, a.parts);
}

int coconet_fused_rs_lamb_ag(coconet_ctx_t c, coconet_tlist_t tl, const void* const* g, int g_elem,
                             float* const* p, float* m_shard, float* v_shard,
                             const coconet_lamb_params* hp, void* stream_) {
  if (!c || !tl || !g || !p || !hp) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  if (tl->ctx != c) return set_error(COCONET_ERR_INVALID_INPUT, "tensor list belongs to another context");
  if (hp->math != COCONET_MATH_FAST && hp->math != COCONET_MATH_EXACT)
    return set_error(COCONET_ERR_INVALID_INPUT, "bad math");
  if (hp->sched < COCONET_LAMB_AUTO || hp->sched > COCONET_LAMB_NVLS)
    return set_error(COCONET_ERR_INVALID_INPUT, "bad LAMB schedule");
  // exchange [rank][tensor] (P, U) doubles + ready flags [rank][tensor]
  if (size_t(kMaxRanks) * tl->n_tensors * (2 * sizeof(double) + sizeof(uint32_t)) > kTileFlagsOff)
    return set_error(COCONET_ERR_UNSUPPORTED, "too many tensors for the exchange area");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int W = c->groups[size_t(tl->group)].size;
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
  k.b1 = double(hp->beta1);
  k.b2 = double(hp->beta2);
  k.c1 = 1.0 - k.b1;
  k.c2 = 1.0 - k.b2;
  k.bc1 = 1.0 - std::pow(k.b1, double(hp->t));
  k.bc2 = 1.0 - std::pow(k.b2, double(hp->t));
  k.eps = double(hp->eps);
  k.wd = double(hp->wd);
  k.guard = hp->trust_guard ? 1 : 0;
  k.csr_ptr = tl->d_csr_ptr;
  k.csr_idx = tl->d_csr_idx;
  k.seg_part = tl->d_seg_part;
  for (int r = 0; r < kMaxRanks; ++r) k.csr_begin[r] = tl->csr_begin[r];
  RankSet rs;
  rc = make_rankset(c, tl->group, &rs);
  if (rc) return rc;
  OptArgs a;
  fill_args(tl, &a, rs, m_off, v_off);
  // AUTO: the TMA ring with buckets of >= kTmaMinBucket elements at W = 1,
  // >= 4x that across ranks (BERT-336M, W = 2/8 virtual: TMA wins at 16384,
  // GRID at 4096; profiles/r01_lamb_w_probe.json), GRID otherwise
  if (hp->math == COCONET_MATH_EXACT && hp->sched == COCONET_LAMB_NVLS)
    return set_error(COCONET_ERR_UNSUPPORTED, "COCONET_LAMB_NVLS runs FAST math (the switch sums in its own order)");
  if (hp->math == COCONET_MATH_EXACT) {  // one schedule: the read-only pass 1 of lamb_exact_kernel
    const void* fn = g_elem == COCONET_F32   ? lamb_exact_pick<float>(W)
                     : g_elem == COCONET_F16 ? lamb_exact_pick<__half>(W)
                                             : lamb_exact_pick<__nv_bfloat16>(W);
    void* args[] = {&a, &k};
    return launch_opt(c, tl, fn, args, false, stream);
  }
  const bool tma_auto = tl->bucket_cap >= (W == 1 ? kTmaMinBucket : 4 * kTmaMinBucket);
  // AUTO at group size 1 with large buckets and a large shard: ONCHIP
  // (BERT-336M: 1.76 ms against TMA's 1.96, profiles/r02_lamb_onchip_probe.json)
  const bool onchip_auto = W == 1 && tma_auto && tl->shard_elems >= kOnchipMinElems;
  const int sched = hp->sched != COCONET_LAMB_AUTO ? hp->sched
                    : onchip_auto                 ? COCONET_LAMB_ONCHIP
                    : tma_auto                    ? COCONET_LAMB_TMA
                                                  : COCONET_LAMB_GRID;
  if (sched == COCONET_LAMB_ONCHIP) {
    if (W != 1) return set_error(COCONET_ERR_UNSUPPORTED, "the ONCHIP LAMB schedule runs at group size 1");
    // consumer warps x quads per thread per chunk item: 16 x 2 (4096-element
    // items, the default), 16 x 1 or 8 x 2 (2048); one CTA per SM
    const char* ne = getenv("COCONET_LAMB_OC_SHAPE");
    const int shape = ne ? atoi(ne) : 162;
    const void* fn = nullptr;
    int sbytes = 0, threads = 0, chunk_q = 0;
    auto pick = [&](auto tag_g) {
      using Gt = decltype(tag_g);
      auto use = [&](auto kern, auto st_tag) {
        using STt = decltype(st_tag);
        fn = reinterpret_cast<const void*>(kern);
        sbytes = STt::BYTES;
        threads = STt::THREADS + 32;  // + the sync warp
        chunk_q = STt::CHUNK_Q;
      };
      if (shape == 161) use(&lamb_onchip_kernel<Gt, 16, 1>, TmaStage<Gt, 16, 1>{});
      else if (shape == 82) use(&lamb_onchip_kernel<Gt, 8, 2>, TmaStage<Gt, 8, 2>{});
      else use(&lamb_onchip_kernel<Gt, 16, 2>, TmaStage<Gt, 16, 2>{});
    };
    if (g_elem == COCONET_F32) pick(float{});
    else if (g_elem == COCONET_F16) pick(__half{});
    else pick(__nv_bfloat16{});
    // one CTA per SM: a ring of S stages, then as many 8 KB u slots as the
    // opt-in shared memory leaves, on top of the 32 TMEM slots
    const char* se = getenv("COCONET_LAMB_OC_STAGES");
    TmaArgs ta;
    int optin = 0, per_sm_smem = 0;
    CN_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
    CN_CUDA(cudaDeviceGetAttribute(&per_sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, c->device));
    cudaFuncAttributes fa;
    CN_CUDA(cudaFuncGetAttributes(&fa, fn));
    // 1 KB per CTA is reserved by the system
    const int budget = std::min(optin, per_sm_smem - 1024) - int(fa.sharedSizeBytes) - 128;
    // the deepest ring that fits (4 stages of 4096-element items at fp16 g:
    // bytes in flight beat shared-memory u slots, profiles/r02_lamb_onchip_probe.json)
    const int fit = std::max(2, std::min(8, budget / (sbytes + 16)));
    ta.stages = se ? std::max(2, std::min(fit, atoi(se))) : std::min(fit, chunk_q == 1024 ? 4 : 5);
    const int slot_off = (ta.stages * sbytes + 16 * ta.stages + 127) / 128 * 128;
    const int room = budget - slot_off;
    const char* xe = getenv("COCONET_LAMB_OC_SMEM_SLOTS");
    const int slot_bytes = chunk_q * 16;  // u of one chunk item
    int smem_slots = std::max(0, room / slot_bytes);
    if (xe) smem_slots = std::max(0, std::min(smem_slots, atoi(xe)));
    LambOC oc;
    oc.tslots = kOcTmemCols / (chunk_q / 32);  // chunk_q * 4 floats over 128 lanes
    oc.cap = oc.tslots + smem_slots;
    const char* he = getenv("COCONET_LAMB_OC_HEAD");
    oc.head = std::max(1, std::min(oc.cap / 2, he ? atoi(he) : 1));
    oc.hold = oc.cap - oc.head;
    if (const char* ke = getenv("COCONET_LAMB_OC_HOLD")) oc.hold = std::max(1, std::min(oc.hold, atoi(ke)));
    const char* h2e = getenv("COCONET_LAMB_OC_HEAD2");
    // one spilled cover item per window by default: it keeps the ring busy
    // while a pass-2 tensor's ratio is still out (-0.7% per step on BERT-336M,
    // profiles/r02_lamb_onchip_head_sweep.txt); its elements re-read m', v'
    oc.head2 = h2e ? std::max(0, std::min(8, atoi(h2e))) : kOcHead2;
    oc.slot_off = slot_off;
    const char* ns = getenv("COCONET_LAMB_OC_NOSYNC");
    oc.nosync = ns ? atoi(ns) : 0;
    const char* tr = getenv("COCONET_LAMB_OC_TRACE");
    oc.trace = tr ? reinterpret_cast<unsigned long long*>(rs.base[0] + atoll(tr)) : nullptr;
    const size_t smem = 128 + size_t(slot_off) + size_t(smem_slots) * slot_bytes;
    rc = ensure_smem(c, fn, smem);
    if (rc) return rc;
    int blocks = 0;
    rc = coop_blocks(c, fn, threads, smem, tl->group, int64_t(c->sm_count), &blocks);
    if (rc) return rc;
    rc = tlist_onchip_plan(tl, blocks, oc.hold, chunk_q, oc.head, oc.head2);
    if (rc) return rc;
    if (tl->oc_K >= 0xffff)
      return set_error(COCONET_ERR_UNSUPPORTED, "ONCHIP LAMB: more than 65534 windows (use the TMA schedule)");
    oc.items = tl->d_oc_items;
    oc.wi = tl->d_oc_wi;
    oc.tfirst = tl->d_oc_tfirst;
    oc.titem = tl->d_oc_titem;
    oc.part = tl->d_oc_part;
    oc.cnt = tl->d_oc_cnt;
    oc.K = tl->oc_K;
    void* args[] = {&a, &k, &ta, &oc};
    return coop_launch(c, fn, dim3(unsigned(blocks), 1u), dim3(unsigned(threads)), args, smem, stream);
  }
  if (sched == COCONET_LAMB_WINDOWED) {
    if (W != 1) return set_error(COCONET_ERR_UNSUPPORTED, "the WINDOWED LAMB schedule runs at group size 1");
    const char* we = getenv("COCONET_LAMB_WIN_ELEMS");
    const int64_t win = hp->lag_elems > 0 ? hp->lag_elems : (we ? atoll(we) : kDefaultWindow);
    rc = tlist_window_plan(tl, win, TmaStage<float, 8, 2>::CHUNK_Q);
    if (rc) return rc;
    const char* ce = getenv("COCONET_LAMB_TMA_CTAS");
    const int per_sm = ce ? std::max(1, std::min(4, atoi(ce))) : 3;
    const void* fn = nullptr;
    int sbytes = 0, threads = 0;
    auto pick = [&](auto tag_g) {
      using Gt = decltype(tag_g);
      using ST = TmaStage<Gt, 8, 2>;
      fn = reinterpret_cast<const void*>(&lamb_win_kernel<Gt, 8, 2>);
      sbytes = ST::BYTES;
      threads = ST::THREADS;
    };
    if (g_elem == COCONET_F32) pick(float{});
    else if (g_elem == COCONET_F16) pick(__half{});
    else pick(__nv_bfloat16{});
    TmaArgs ta;
    ta.stages = std::min(16, (200 << 10) / per_sm / sbytes);
    if (ta.stages < 2) return set_error(COCONET_ERR_UNSUPPORTED, "TMA ring does not fit");
    const size_t smem = size_t(ta.stages) * size_t(sbytes) + size_t(ta.stages) * 16 + 128;
    rc = ensure_smem(c, fn, smem);
    if (rc) return rc;
    int blocks = 0;
    rc = coop_blocks(c, fn, threads, smem, tl->group, int64_t(c->sm_count) * per_sm, &blocks);
    if (rc) return rc;
    if (ta.stages > 16) ta.stages = 16;
    LambWin lw;
    lw.items = tl->d_win_items;
    lw.wi = tl->d_win_item;
    lw.titem = tl->d_titem;
    lw.tfirst = tl->d_win_t;
    lw.tick = tl->d_win_tick;
    lw.cnt = tl->d_win_cnt;
    lw.ready = tl->d_win_ready;
    lw.ipart = tl->d_ipart;
    lw.ratio = tl->d_ratio;
    lw.K = tl->n_windows;
    // tickets, arrivals and ready flags are cumulative over calls (no reset
    // kernel): restart them when the grid size changes
    if (tl->win_blocks != blocks) {
      CN_CUDA(cudaMemsetAsync(tl->win_state, 0, tl->win_state_bytes, stream));
      tl->win_blocks = blocks;
      tl->win_calls = 0;
    }
    lw.call = ++tl->win_calls;
    const char* he = getenv("COCONET_LAMB_WIN_HEAD");
    lw.head = int64_t(he ? std::max(0, atoi(he)) : 2) * blocks * kWinBatch;
    void* args[] = {&a, &k, &ta, &lw};
    return coop_launch(c, fn, dim3(unsigned(blocks), 1u), dim3(unsigned(threads)), args, smem, stream);
  }
  if (sched == COCONET_LAMB_TMA) {
    // 8 consumer warps x 2 quads per thread (2048-element chunks), 3 CTAs
    // per SM: the best of the sweep in profiles/r01_lamb_tma_sweep.json
    // (COCONET_LAMB_TMA_CTAS overrides the CTAs per SM the ring is sized
    // for). Registers keep 2 resident, so this is a 2-stage ring of 2048-
    // element chunks, which also measured best at W = 2/4/8
    // (profiles/r01_lamb_w_probe.json: a 3-stage ring is 1-4% slower).
    const char* ce = getenv("COCONET_LAMB_TMA_CTAS");
    const int per_sm = ce ? std::max(1, std::min(4, atoi(ce))) : 3;
    const void* fn = nullptr;
    int sbytes = 0, threads = 0;
    auto pick = [&](auto tag_g) {
      using Gt = decltype(tag_g);
      using ST = TmaStage<Gt, 8, 2>;
      fn = W == 1   ? reinterpret_cast<const void*>(&lamb_tma_kernel<Gt, 8, 2, 1>)
           : W == 2 ? reinterpret_cast<const void*>(&lamb_tma_kernel<Gt, 8, 2, 2>)
           : W == 4 ? reinterpret_cast<const void*>(&lamb_tma_kernel<Gt, 8, 2, 4>)
           : W == 8 ? reinterpret_cast<const void*>(&lamb_tma_kernel<Gt, 8, 2, 8>)
                    : reinterpret_cast<const void*>(&lamb_tma_kernel<Gt, 8, 2, 0>);
      sbytes = ST::BYTES;
      threads = ST::THREADS;
    };
    if (g_elem == COCONET_F32) pick(float{});
    else if (g_elem == COCONET_F16) pick(__half{});
    else pick(__nv_bfloat16{});
    TmaArgs ta;
    ta.stages = std::min(16, (200 << 10) / per_sm / sbytes);
    if (ta.stages < 2) return set_error(COCONET_ERR_UNSUPPORTED, "TMA ring does not fit");
    const size_t smem = size_t(ta.stages) * size_t(sbytes) + size_t(ta.stages) * 16 + 128;
    rc = ensure_smem(c, fn, smem);
    if (rc) return rc;
    int blocks = 0;
    const int lr = local_ranks(c, tl->group);
    rc = coop_blocks(c, fn, threads, smem, tl->group, int64_t(c->sm_count) * per_sm / lr, &blocks);
    if (rc) return rc;
    void* args[] = {&a, &k, &ta};
    return coop_launch(c, fn, dim3(unsigned(blocks), unsigned(lr)), dim3(unsigned(threads)), args, smem, stream);
  }
  if (sched == COCONET_LAMB_NVLS) {
    if (!c->mc_base || tl->group != 0)
      return set_error(COCONET_ERR_UNSUPPORTED, "COCONET_LAMB_NVLS needs coconet_nvls_setup on the world group "
                                                "(coconet_nvls_supported reports why it is unavailable)");
    const void* fn = g_elem == COCONET_F32   ? reinterpret_cast<const void*>(&lamb_kernel<float, 0, 2, true>)
                     : g_elem == COCONET_F16 ? reinterpret_cast<const void*>(&lamb_kernel<__half, 0, 2, true>)
                                             : reinterpret_cast<const void*>(&lamb_kernel<__nv_bfloat16, 0, 2, true>);
    void* args[] = {&a, &k};
    return launch_opt(c, tl, fn, args, false, stream);
  }
  if (sched == COCONET_LAMB_GRID) {
    const void* fn = g_elem == COCONET_F32   ? lamb_pick<float>(W)
                     : g_elem == COCONET_F16 ? lamb_pick<__half>(W)
                                             : lamb_pick<__nv_bfloat16>(W);
    void* args[] = {&a, &k};
    return launch_opt(c, tl, fn, args, false, stream);
  }
  // STREAMED (default)
  const int64_t lag = hp->lag_elems > 0 ? hp->lag_elems : kDefaultLag;
  rc = tlist_stream_plan(tl, lag);
  if (rc) return rc;
  LambS ls;
  ls.items = tl->d_items;
  ls.p1_first = tl->d_p1_first;
  ls.holders = tl->d_holders;
  ls.cnt = tl->d_cnt;
  ls.part = tl->d_item_part;
  for (int r = 0; r <= kMaxRanks; ++r) ls.item_begin[r] = r <= W ? tl->item_begin[r] : 0;
  ls.rdy_off = int64_t(kMaxRanks) * tl->n_tensors * 2 * int64_t(sizeof(double));
  ls.call = ++tl->stream_calls;
  const void* fn = g_elem == COCONET_F32   ? lamb_stream_pick<float>(W)
                   : g_elem == COCONET_F16 ? lamb_stream_pick<__half>(W)
                                           : lamb_stream_pick<__nv_bfloat16>(W);
  void* args[] = {&a, &k, &ls};
  int64_t most = 0;
  for (int r = 0; r < W; ++r) most = std::max(most, tl->item_begin[r + 1] - tl->item_begin[r]);
  int blocks = 0;
  const int nt = W == 1 ? 64 : (W == 2 || W == 4) ? 128 : 256;  // lamb_stream_pick's CTA sizes
  rc = coop_blocks(c, fn, nt, 0, tl->group, most, &blocks);
  if (rc) return rc;
  return coop_launch(c, fn, dim3(unsigned(blocks), unsigned(local_ranks(c, tl->group))), dim3(unsigned(nt)),
                     args, 0, stream);
}

int coconet_allreduce(coconet_ctx_t c, coconet_tlist_t tl, const void* const* x, void* const* out,
                      int elem, int reducer, int algo, void* stream_) {
  if (!c || !tl || !x || !out) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  if (tl->ctx != c) return set_error(COCONET_ERR_INVALID_INPUT, "tensor list belongs to another context");
  if (elem < COCONET_F32 || elem > COCONET_BF16) return set_error(COCONET_ERR_INVALID_INPUT, "bad elem");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int W = c->groups[size_t(tl->group)].size;
  const bool nvls = algo == COCONET_ALGO_NVLS;
  if (nvls && (!c->mc_base || tl->group != 0))
    return set_error(COCONET_ERR_UNSUPPORTED, "COCONET_ALGO_NVLS needs coconet_nvls_setup on the world group "
                                              "(coconet_nvls_supported reports why it is unavailable)");
  if (nvls && reducer != COCONET_SUM)
    return set_error(COCONET_ERR_UNSUPPORTED, "COCONET_ALGO_NVLS reduces with SUM only");
  bool os = !nvls && resolve_one_shot(algo, tl, W);
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
  const void* fn = nvls ? (elem == COCONET_F32   ? reinterpret_cast<const void*>(&allreduce_nvls_kernel<float>)
                           : elem == COCONET_F16 ? reinterpret_cast<const void*>(&allreduce_nvls_kernel<__half>)
                                                 : reinterpret_cast<const void*>(&allreduce_nvls_kernel<__nv_bfloat16>))
                   : elem == COCONET_F32 ? ar_pick<float>(reducer, os, W)
                   : elem == COCONET_F16 ? ar_pick<__half>(reducer, os, W)
                                         : ar_pick<__nv_bfloat16>(reducer, os, W);
  void* args[] = {&a};
  return launch_opt(c, tl, fn, args, os, stream);
}

}  // extern "C"
