// MatMul for the model-parallel pattern (goldens/model_parallel.json: the
// row-parallel layer [B,S,H/W] x [H/W,H] -> Local partial sums), and its
// overlap with the fused AllReduce epilogue (schedules/mp_overlap.json:
// OverlapGroup{MatMul, FusedAllReduce}).
//
// Reference: eval_matmul (state.hpp:94-121) computes per rank the K-slice
// partial product with double accumulation; OverlapGroup (runtime.hpp:517-522)
// runs its members sequentially and only its simulated clock overlaps them
// (overlap_time :230-271, tile order chunk_order :46-50).
//
// B200:
//  * FAST (bf16/fp16 inputs): a persistent warp-specialised tcgen05 kernel.
//    Warp 0 issues TMA loads (128B-swizzled K-major tiles) into a 4-stage
//    smem ring guarded by mbarriers; warp 1 (one elected thread) issues
//    tcgen05.mma (M=128, N=BN, K=16) into a double-buffered TMEM accumulator;
//    warps 4-7 drain TMEM with tcgen05.ld, convert, store the tile and — for
//    the overlap — publish a per-tile flag (st.release.sys) that the
//    communication kernel of every rank polls.
//  * EXACT (fp32 inputs): fp64 accumulation in k order on the FP64 pipe,
//    bit-identical to eval_matmul (each fp32*fp32 product is exact in double,
//    so FMA == multiply-then-add).
//  * Overlap (one cooperative kernel, 16 warps per CTA): warps 2, 3 and 8-15
//    start on the all-reduce at once, warps 0/1/4-7 join when their GEMM roles
//    finish. A unit (row tile, owner rank, 32 rows) is taken from an atomic
//    ticket in row-tile order and starts as soon as every rank has published
//    the tiles it covers, so the RS -> bias+dropout+residual -> AG of row tile
//    i overlaps the MMAs of later row tiles. GEMM warps never wait on comm
//    warps, so the kernel cannot deadlock.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>

#include "internal.h"
#include "pipeline.cuh"

using namespace coconet;

namespace {

constexpr int BM = 128, BK = 64;
constexpr int kGemmThreads = 256;
constexpr int kAccStride = 256;   // TMEM columns per accumulator buffer
constexpr int kTmemCols = 512;
constexpr int kFusedThreads = 512;  // overlap kernel: 16 warps (0/1/4-7 GEMM roles, the rest all-reduce)
constexpr int kFusedWarps = kFusedThreads / 32;

// Stage counts: the K=384 GEMM is bound by TMA bytes in flight, so the ring
// takes all the shared memory the epilogue leaves (4 x 48 KB at BN = 256;
// 3 stages: 193 us for C3's 8 ranks, 4 stages: 172 us).
template <int BN> struct Cfg {
  static constexpr int STAGES = 4;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_BYTES = 4 * 2 * 4096;  // 4 epilogue warps x 2 staging buffers of 32 rows x 128 B
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 256;
};

struct RankMaps {
  CUtensorMap a[kMaxRanks];
  CUtensorMap a_half[kMaxRanks];  // 64-row boxes: the multicast halves of A (MC)
  CUtensorMap b[kMaxRanks];
  CUtensorMap c[kMaxRanks];  // output, stored by TMA from swizzled staging tiles
};

struct GemmArgs {
  char* c[kMaxRanks];          // C (row-major [M, N]) of each rank computed here
  uint32_t* flags[kMaxRanks];  // per-tile flags of each rank (nullable)
  int M, N, K;
  int ranks;                   // ranks computed by this launch
  int tiles_m, tiles_n;
  uint32_t epoch;
  int local_peers;             // every rank on this GPU (VIRTUAL): flags need only gpu scope
  int diag;                    // COCONET_GEMM_DIAG (profiling only): 1 = no C stores, 2 = no A/B loads
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// TMA load multicast to every CTA of the cluster in `mask` (same smem offset
// and the barrier at the same offset in each destination CTA).
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major operand tile [rows x 64] bf16 with 128-byte swizzle (as TMA writes
// it): 8-row atoms of 1024 B; LBO unused (1), SBO = 1024 B, version 1.
__device__ __forceinline__ uint64_t sw128_desc(const void* p) {
  const uint64_t addr = smem_u32(p);
  return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// MN-major operand tile [64 k x BN] bf16 loaded as BN/64 TMA boxes of
// [64 k rows x 64 n] (128-byte swizzle, 1 KB per 8 k-rows): the canonical
// UMMA MN-major SW128 layout ((T,8,m),(8,k)) : ((1,T,LBO),(8T,SBO)) with
// LBO = 8 KB (next 64 n) and SBO = 1 KB (next 8 k), version 1 (CUTLASS
// make_umma_desc<Major::MN>). B is read in its natural row-major [K, N]
// layout: no transpose.
constexpr int kMnBlockBytes = 64 * 64 * 2;
__device__ __forceinline__ uint64_t sw128_mn_desc(const void* p) {
  const uint64_t addr = smem_u32(p);
  return ((addr >> 4) & 0x3FFFull) | (uint64_t(kMnBlockBytes >> 4) << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// arrive on `bar` in both CTAs of a 2-CTA cluster once these MMAs retire
__device__ __forceinline__ void mma_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// instruction descriptor: kind::f16, A/B = in_fmt (0 f16, 1 bf16), D = f32,
// A K-major, B MN-major (bit 16), M = 128, N = BN
template <int BN>
__device__ __forceinline__ uint32_t make_idesc(uint32_t in_fmt) {
  return (1u << 4) | (in_fmt << 7) | (in_fmt << 10) | (1u << 16) | (uint32_t(BN >> 3) << 17) |
         (uint32_t(BM >> 4) << 24);
}

template <typename TO>
__device__ __forceinline__ void store_row32(TO* dst, const uint32_t (&v)[32]) {
  if constexpr (sizeof(TO) == 4) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      reinterpret_cast<uint4*>(dst)[i] = make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  } else {
    uint32_t h[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      TO lo = from_f32<TO>(__uint_as_float(v[2 * i]));
      TO hi = from_f32<TO>(__uint_as_float(v[2 * i + 1]));
      h[i] = uint32_t(*reinterpret_cast<uint16_t*>(&lo)) | (uint32_t(*reinterpret_cast<uint16_t*>(&hi)) << 16);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      reinterpret_cast<uint4*>(dst)[i] = make_uint4(h[4 * i], h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
  }
}

// Tile flag: release at gpu scope when every reader is on this GPU
// (VIRTUAL), at system scope when peers read over NVLink.
__device__ __forceinline__ void publish_flag(uint32_t* f, uint32_t epoch, int local) {
  if (local) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
  } else {
    __threadfence_system();
    st_release_sys(f, epoch);
  }
}

// Tile order: row tiles outermost, then column tiles, then ranks, so every
// rank publishes row tile i of every column block before row tile i+1 and the
// consumers of all column blocks can start together.
__device__ __forceinline__ void decode_tile(const GemmArgs& g, int t, int& r, int& mt, int& nt) {
  const int per_m = g.tiles_n * g.ranks;
  mt = t / per_m;
  const int j = t - mt * per_m;
  nt = j / g.ranks;
  r = j - nt * g.ranks;
}

// MC: tile t of the pair sequence. MC == 1 (A shared): CTA crank of the
// cluster takes column tile 2j + crank of a row tile; MC == 2 (B shared): row
// tile 2i + crank of a column tile.
template <int MC>
__device__ __forceinline__ void decode_tile2(const GemmArgs& g, int t, uint32_t crank, int& r, int& mt, int& nt) {
  if constexpr (MC == 1) {
    const int per_m = (g.tiles_n / 2) * g.ranks;
    mt = t / per_m;
    const int j = t - mt * per_m;
    const int np = j / g.ranks;
    r = j - np * g.ranks;
    nt = 2 * np + int(crank);
  } else if constexpr (MC == 2) {
    const int per_m = g.tiles_n * g.ranks;
    const int mp = t / per_m;
    const int j = t - mp * per_m;
    nt = j / g.ranks;
    r = j - nt * g.ranks;
    mt = 2 * mp + int(crank);
  } else {
    decode_tile(g, t, r, mt, nt);
  }
}

// ---- fused all-reduce epilogue of the overlapped MatMul (mp_overlap.json) ----
// Work unit = (row tile mt, owner rank, 32-row group): one warp pulls that
// block of column block `owner` from every rank's partial sums (ring-order
// fp32 fold), applies dropout(x + b) + r and pushes it into every rank's out.
// Units are handed out in row-tile order by an atomic ticket, so the earliest
// tiles the GEMM publishes are reduced first.
struct OvArgs {
  RankSet rs;            // group ranks (peer heaps), epoch of this call
  int64_t part_off, b_off, r_off, out_off;
  int64_t cnt_off;       // per-rank arrival counter (uint32) in the reserved area
  int64_t flag_off;      // per-rank tile flags
  int64_t ticket_off;    // unit ticket counter (in the first local rank's heap)
  int rows, cols, per;   // per = cols / W
  int tiles_m, tiles_n, bn;
  int nl;                // local ranks of this launch
  int n_units;           // tiles_m * nl * 4
  uint32_t ticket_base;  // ticket value at the start of this call
  uint32_t arrive_target;  // cumulative arrivals expected on each rank's counter
  double inv_keep;
  float frate_scale;
  uint64_t seed, key, thresh;
  int math;
};

// One unit = 32 rows of column block `me`; each lane moves MP_U 16-byte
// vectors (V = 8 16-bit elements) per rank per step, with every rank's
// vectors, b and r in flight before the ring-order fold (the comm region may
// use the registers the GEMM epilogue already holds).
#ifndef MP_U
#define MP_U 2
#endif
template <typename T>
__device__ __forceinline__ void mp_unit(const OvArgs& a, char* const* base, int me, int mt, int rg, int lane) {
  static_assert(sizeof(T) == 2, "the overlapped all-reduce moves 16-bit partials");
  constexpr int V = 8, U = MP_U;
  const int W = a.rs.world;
  const int vpr = a.per / V;  // vectors per row of the block
  const int nv = 32 * vpr;
  for (int i0 = lane; i0 < nv; i0 += 32 * U) {
    int64_t gi[U];
    uint4 raw[U][kMaxRanks], braw[U], rraw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = min(i0 + 32 * u, nv - 1);  // clamped, unconditional loads
      const int row = mt * 128 + rg * 32 + i / vpr;
      gi[u] = int64_t(row) * a.cols + int64_t(me) * a.per + (i % vpr) * V;
#pragma unroll
      for (int j = 0; j < kMaxRanks; ++j)
        if (j < W) {
          int src = me + 1 + j;
          src -= src >= W ? W : 0;
          src -= src >= W ? W : 0;
          raw[u][j] = __ldcg(reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(base[src] + a.part_off) + gi[u]));
        }
      braw[u] = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(base[me] + a.b_off) + gi[u] % a.cols));
      rraw[u] = __ldcg(reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(base[me] + a.r_off) + gi[u]));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i0 + 32 * u >= nv) break;
      uint4 ov;
      T* o = reinterpret_cast<T*>(&ov);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        float acc = to_f32(reinterpret_cast<const T*>(&raw[u][0])[e]);
#pragma unroll
        for (int j = 1; j < kMaxRanks; ++j)
          if (j < W) acc = __fadd_rn(acc, to_f32(reinterpret_cast<const T*>(&raw[u][j])[e]));
        const float bv = to_f32(reinterpret_cast<const T*>(&braw[u])[e]);
        const float rv = to_f32(reinterpret_cast<const T*>(&rraw[u])[e]);
        const bool keep = dropout_keep_bits(a.seed, a.key, uint64_t(gi[u] + e), a.thresh);
        float y;
        if (a.math == COCONET_MATH_EXACT) {
          const double sum = __dadd_rn(double(acc), double(bv));
          y = float(__dadd_rn(keep ? __ddiv_rn(sum, a.inv_keep) : 0.0, double(rv)));
        } else {
          y = (keep ? (acc + bv) * a.frate_scale : 0.f) + rv;
        }
        o[e] = from_f32<T>(y);
      }
#pragma unroll
      for (int j = 0; j < kMaxRanks; ++j) {
        if (j >= W) break;
        *reinterpret_cast<uint4*>(reinterpret_cast<T*>(base[j] + a.out_off) + gi[u]) = ov;
      }
    }
  }
}

// Tile-flag wait of a comm unit: the unit usually waits for tiles the GEMM
// publishes microseconds later, so it polls with relaxed loads (an acquire
// load invalidates L1 every poll) and backs off exponentially up to 2 us,
// keeping ~1.5k waiting warps from flooding L2 next to the GEMM's TMA
// traffic; one acquire fence orders the partial-sum reads after the flag.
__device__ __forceinline__ bool wait_tile_flag(const uint32_t* p, uint32_t want, const RankSet& rs, bool local) {
  uint32_t v;
  if (local)
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  if (int32_t(v - want) < 0) {
    const unsigned long long t0 = globaltimer();
    unsigned ns = 128;
    for (;;) {
      __nanosleep(ns);
      ns = ns < 2048 ? ns * 2 : 2048;
      if (local)
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
      else
        asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
      if (int32_t(v - want) >= 0) break;
      if (globaltimer() - t0 > rs.timeout_ns) {
        atomicCAS(rs.status, 0, COCONET_ERR_TIMEOUT);
        return false;
      }
    }
  }
  return true;
}

// One warp's share of the all-reduce: take tickets until the units run out.
template <typename T>
__device__ void mp_comm_warp(const OvArgs& a, char* const* base, int lane) {
  const unsigned full = 0xffffffffu;
  const int W = a.rs.world;
  unsigned int* ticket = reinterpret_cast<unsigned int*>(base[a.rs.me >= 0 ? a.rs.me : 0] + a.ticket_off);
  for (;;) {
    int u = 0;
    if (lane == 0) u = int(atomicAdd(ticket, 1u) - a.ticket_base);
    u = __shfl_sync(full, u, 0);
    if (u < 0 || u >= a.n_units) break;  // u < 0: the ticket counter is behind ticket_base
    const int mt = u / (a.nl * 4);
    const int rem = u - mt * a.nl * 4;
    const int lr = rem >> 2, rg = rem & 3;
    const int me = a.rs.me >= 0 ? a.rs.me : lr;
    const int t_lo = (me * a.per) / a.bn, t_hi = ((me + 1) * a.per - 1) / a.bn;
    // VIRTUAL (every rank in this grid): gpu-scope flags, fences and
    // arrivals; across processes, system scope. One acquire fence per lane
    // after all its flags.
    const bool local = a.rs.me < 0;
    bool ok = true;
    if (lane < W) {
      const uint32_t* fl = reinterpret_cast<const uint32_t*>(base[lane] + a.flag_off);
      for (int nt = t_lo; nt <= t_hi; ++nt) ok &= wait_tile_flag(fl + mt * a.tiles_n + nt, a.rs.epoch, a.rs, local);
      if (local)
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      else
        asm volatile("fence.acq_rel.sys;" ::: "memory");
    }
    if (!__all_sync(full, ok)) continue;  // watchdog fired; status already recorded
    mp_unit<T>(a, base, me, mt, rg, lane);
    __syncwarp();
    if (lane < W) {  // one arrival per (unit, destination rank)
      if (local) {
        __threadfence();
        atomicAdd(reinterpret_cast<unsigned int*>(base[lane] + a.cnt_off), 1u);
      } else {
        __threadfence_system();
        atomicAdd_system(reinterpret_cast<unsigned int*>(base[lane] + a.cnt_off), 1u);
      }
    }
  }
}

// MC (plain GEMM only): clusters of 2 CTAs share one operand tile by TMA
// multicast, each CTA loading half of it into both CTAs' smem.
//   MC == 1: column tiles 2j and 2j+1 of one row tile share A (64-row halves);
//   MC == 2: row tiles 2i and 2i+1 of one column tile share B (BN/2-column
//            halves): B is the larger operand (BN = 256 > BM = 128), so this
//            halves more L2 -> SM traffic.
// The stage barriers then count both CTAs' MMAs (either CTA's producer writes
// into both CTAs' stages).
template <int BN, typename TO, bool FUSED, int MC>
__global__ void __launch_bounds__(FUSED ? kFusedThreads : kGemmThreads, 1)
    gemm_tc_kernel(const __grid_constant__ RankMaps maps, GemmArgs g, uint32_t in_fmt, OvArgs ov) {
  static_assert(!(MC && FUSED), "multicast is for the plain GEMM");
  __shared__ char* s_base[kMaxRanks];
  if (FUSED && threadIdx.x < kMaxRanks)
    s_base[threadIdx.x] = threadIdx.x < ov.rs.world ? ov.rs.base[threadIdx.x] : nullptr;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi = smem + Cfg<BN>::STAGES * Cfg<BN>::STAGE_BYTES;  // 1024-aligned staging
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + Cfg<BN>::EPI_BYTES);
  uint64_t* empty = full + Cfg<BN>::STAGES;
  uint64_t* tfull = empty + Cfg<BN>::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < Cfg<BN>::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC ? 2 : 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (MC) cluster_sync();  // the peer multicasts into our barriers: they must exist
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t crank = MC ? cluster_ctarank() : 0u;
  // MC: the cluster walks pair tiles (column tiles 2j, 2j+1), CTA crank takes 2j + crank
  const int total = MC == 1   ? g.ranks * g.tiles_m * (g.tiles_n / 2)
                    : MC == 2 ? g.ranks * (g.tiles_m / 2) * g.tiles_n
                              : g.ranks * g.tiles_m * g.tiles_n;
  const int tile0 = MC ? int(blockIdx.x >> 1) : int(blockIdx.x);
  const int tstride = MC ? int(gridDim.x >> 1) : int(gridDim.x);
  const int kblocks = g.K / BK;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = tile0; t < total; t += tstride) {
        int r, mt, nt;
        decode_tile2<MC>(g, t, crank, r, mt, nt);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg<BN>::STAGE_BYTES;
          if (g.diag & 2) {
            mbar_arrive(&full[stage]);
            if (++stage == Cfg<BN>::STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          mbar_expect_tx(&full[stage], Cfg<BN>::STAGE_BYTES);
          if constexpr (MC == 1)  // our 64-row half of A into both CTAs
            tma_load_2d_mc(sa + crank * (Cfg<BN>::A_BYTES / 2), &maps.a_half[r], kb * BK,
                             mt * BM + int(crank) * 64, &full[stage], uint16_t(3));
          else
            tma_load_2d(sa, &maps.a[r], kb * BK, mt * BM, &full[stage]);
#pragma unroll
          for (int j = 0; j < BN / 64; ++j) {  // B [K, N] row-major: 64 n x 64 k boxes
            if constexpr (MC == 2) {  // our half of the boxes into both CTAs
              if (j / (BN / 128) == int(crank))
                tma_load_2d_mc(sa + Cfg<BN>::A_BYTES + j * kMnBlockBytes, &maps.b[r], nt * BN + j * 64, kb * BK,
                                 &full[stage], uint16_t(3));
            } else {
              tma_load_2d(sa + Cfg<BN>::A_BYTES + j * kMnBlockBytes, &maps.b[r], nt * BN + j * 64, kb * BK,
                            &full[stage]);
            }
          }
          if (++stage == Cfg<BN>::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    if constexpr (FUSED) {
      __syncwarp();
      mp_comm_warp<TO>(ov, s_base, lane);
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer (single thread)
      const uint32_t idesc = make_idesc<BN>(in_fmt);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = tile0; t < total; t += tstride) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + uint32_t(acc * kAccStride);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint8_t* sa = smem + stage * Cfg<BN>::STAGE_BYTES;
          const uint64_t da = sw128_desc(sa), db = sw128_mn_desc(sa + Cfg<BN>::A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)  // per UMMA_K = 16: A +32 bytes along K, B +16 k-rows (2 KB)
            mma_f16(d, da + 2 * k, db + uint64_t(k) * ((16 * 128) >> 4), idesc, (kb | k) != 0);
          if constexpr (MC)
            mma_commit_both(&empty[stage]);  // both CTAs' producers write into this stage
          else
            mma_commit(&empty[stage]);  // frees the smem stage once these MMAs retire
          if (++stage == Cfg<BN>::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[acc]);  // accumulator complete -> epilogue
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
    if constexpr (FUSED) {
      __syncwarp();
      mp_comm_warp<TO>(ov, s_base, lane);
    }
  } else if (warp >= 4 && warp < 8) {  // ---- epilogue: TMEM -> registers -> swizzled smem -> TMA store
    const int q = warp & 3;
    uint8_t* stg = epi + q * 2 * 4096;
    constexpr int kCols = 128 / int(sizeof(TO));  // columns per 128-byte row chunk
    int acc = 0, buf = 0;
    uint32_t acc_phase = 0;
    uint32_t* pend_flag = nullptr;  // tile flag published once its stores are complete
    for (int t = tile0; t < total; t += tstride) {
      int r, mt, nt;
      decode_tile2<MC>(g, t, crank, r, mt, nt);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem + (uint32_t(q * 32) << 16) + uint32_t(acc * kAccStride);
#pragma unroll 1
      for (int cc = 0; cc < BN / kCols; ++cc) {
        // this staging buffer was last read by the store issued two chunks ago
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        uint8_t* row = stg + buf * 4096 + lane * 128;
        uint32_t h[32];
        if constexpr (sizeof(TO) == 4) {
          uint32_t v[32];
          tmem_ld32(tbase + uint32_t(cc * 32), v);
#pragma unroll
          for (int i = 0; i < 32; ++i) h[i] = v[i];
        } else {
          uint32_t v[32], w[32];
          tmem_ld32(tbase + uint32_t(cc * 64), v);
          tmem_ld32(tbase + uint32_t(cc * 64 + 32), w);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            TO lo = from_f32<TO>(__uint_as_float(v[2 * i])), hi = from_f32<TO>(__uint_as_float(v[2 * i + 1]));
            h[i] = uint32_t(*reinterpret_cast<uint16_t*>(&lo)) | (uint32_t(*reinterpret_cast<uint16_t*>(&hi)) << 16);
            TO lo2 = from_f32<TO>(__uint_as_float(w[2 * i])), hi2 = from_f32<TO>(__uint_as_float(w[2 * i + 1]));
            h[16 + i] =
                uint32_t(*reinterpret_cast<uint16_t*>(&lo2)) | (uint32_t(*reinterpret_cast<uint16_t*>(&hi2)) << 16);
          }
        }
        if (g.diag & 1) {
          if (h[0] == 0x7fffffffu && h[31] == 0x7fffffffu) g.c[0][0] = 1;  // keep the loads live
          continue;
        }
        // 128B swizzle (matches the output tensor map): chunk j of row l lands at j ^ (l % 8)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint4*>(row + ((j ^ (lane & 7)) << 4)) = make_uint4(h[4 * j], h[4 * j + 1], h[4 * j + 2], h[4 * j + 3]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&maps.c[r], stg + buf * 4096, nt * BN + cc * kCols, mt * BM + q * 32);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        buf ^= 1;
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (g.flags[r] != nullptr) {
        // publish the PREVIOUS tile's flag: only its store groups (all but
        // this tile's BN / kCols) must be complete, so the epilogue never
        // waits for the stores it just issued
        if (pend_flag) {
          if (lane == 0) {
            asm volatile("cp.async.bulk.wait_group %0;" ::"n"(BN / kCols) : "memory");
            asm volatile("fence.proxy.async;" ::: "memory");
          }
          __syncwarp();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (warp == 4 && lane == 0) publish_flag(pend_flag, g.epoch, g.local_peers);
        }
        pend_flag = g.flags[r] + mt * g.tiles_n + nt;
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
    if (pend_flag) {  // the last tile
      if (lane == 0) asm volatile("fence.proxy.async;" ::: "memory");
      __syncwarp();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (warp == 4 && lane == 0) publish_flag(pend_flag, g.epoch, g.local_peers);
    }
    if constexpr (FUSED) mp_comm_warp<TO>(ov, s_base, lane);
  } else if constexpr (FUSED) {  // warps 2, 3 and 8-15: all-reduce from the start
    mp_comm_warp<TO>(ov, s_base, lane);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (MC) cluster_sync();  // no CTA leaves while its peer may still multicast into it
  tc_fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  // the caller's `out` is complete once every unit of every owner has landed
  if (FUSED && blockIdx.x == 0 && threadIdx.x < ov.nl) {
    const int r = ov.rs.me >= 0 ? ov.rs.me : int(threadIdx.x);
    wait_flag(reinterpret_cast<const uint32_t*>(s_base[r] + ov.cnt_off), ov.arrive_target, ov.rs);
  }
}

// ---- 2-SM pair GEMM with the B panel resident (plain GEMM, BN = 256) ----
// At K = 384 a 128 x 256 tile is 25 MFLOP against 288 KB of A and B through
// L2 -> SM (15.7 TB/s over the chip at the tensor peak); the operand loads
// and the C stores together cost ~50 us over the MMAs (profiles/r01_gemm_diag.json).
// Here two CTAs of a cluster run tcgen05.mma.cta_group::2 (M = 256, N = 256):
// each CTA holds 128 rows of A and 128 columns of B and receives its 128 rows
// x 256 columns of D in its own TMEM. B stays RESIDENT in shared memory for a
// whole (rank, column block) panel (K x 128 bf16 = 96 KB at K = 384), so only
// A streams: 96 KB per 2 x 25 MFLOP, 2.5x less L2 -> SM traffic.
//   warp 0   producer (each CTA): B half panel on a panel change, A k-blocks
//            into a 4-stage ring; both CTAs' loads complete on the LEADER's
//            barriers (cp.async.bulk.tensor .cta_group::2)
//   warp 1   MMA issuer (leader only); commits multicast to both CTAs
//   warp 2   TMEM allocator (cta_group::2, both CTAs)
//   warps 4-7 epilogue (each CTA): TMEM -> bf16 -> swizzled smem -> TMA store;
//            one remote arrive per CTA on the leader's accumulator-empty barrier
// Work: units (rank, 256-column block = panel, 256-row block). Pairs take
// whole panels in rounds (pair p: panels p, p + P, ...) and walk their row
// blocks in step, so the ~P/ranks pairs on one rank read the same A row block
// at the same time (one DRAM read, L2 hits for the rest); the panels left
// over after the last full round are split into equal unit ranges.
constexpr int kPairMaxStages = 8;
constexpr int kPairABytes = BM * BK * 2;       // 16 KB: 128 rows x 64 k
constexpr int kPairBBytes = 2 * kMnBlockBytes;  // 16 KB per k-block: 2 boxes of 64 n x 64 k
#ifndef COCONET_PAIR_EPI_BUFS
#define COCONET_PAIR_EPI_BUFS 2
#endif
constexpr int kPairEpiBufs = COCONET_PAIR_EPI_BUFS;  // staging buffers per epilogue warp (4 KB each)
constexpr int kPairEpiBytes = 4 * kPairEpiBufs * 4096;
constexpr int kPairKMax = 512;

// A stages: what the shared memory leaves after the B panel and the staging
__host__ __device__ constexpr int pair_stages(int kblocks) {
  return (227 * 1024 - kblocks * kPairBBytes - kPairEpiBytes - 1024 - 512) / kPairABytes < kPairMaxStages
             ? (227 * 1024 - kblocks * kPairBBytes - kPairEpiBytes - 1024 - 512) / kPairABytes
             : kPairMaxStages;
}
__host__ __device__ constexpr int pair_smem(int kblocks) {
  return kblocks * kPairBBytes + pair_stages(kblocks) * kPairABytes + kPairEpiBytes + 1024 + 512;
}

__device__ __forceinline__ uint32_t mapa_leader(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
// Arrive on a barrier of either pair CTA (release at CTA scope, as CUTLASS's
// ClusterBarrier::arrive(cta_id): .release.cluster compiles to a MEMBAR.ALL.GPU
// per arrive, which serialised the producer)
__device__ __forceinline__ void mbar_arrive_cl(uint32_t cl_bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cl_bar) : "memory");
}
// TMA load into this CTA's smem completing on a barrier of either pair CTA,
// with an L2 eviction policy
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1, uint32_t cl_bar,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(cl_bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, const void* src, int c0, int c1,
                                                  uint64_t policy) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(smem_u32(src)), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void mma_f16_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// arrive on `bar` (same offset) in both pair CTAs once the pair MMAs issued so far retire
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}

// M = 256 (pair), N = 256, A K-major, B MN-major
__device__ __forceinline__ uint32_t make_idesc_pair(uint32_t in_fmt) {
  return (1u << 4) | (in_fmt << 7) | (in_fmt << 10) | (1u << 16) | (uint32_t(256 >> 3) << 17) |
         (uint32_t(256 >> 4) << 24);
}

struct PairSched {
  int P, p, mbs, np, rounds, lu0, lu1;
  __device__ __forceinline__ PairSched(const GemmArgs& g, int pairs, int pair) : P(pairs), p(pair) {
    mbs = g.tiles_m / 2;  // 256-row blocks
    np = g.ranks * g.tiles_n;
    rounds = np / P;
    const int left = (np - rounds * P) * mbs;
    lu0 = int(int64_t(left) * p / P);
    lu1 = int(int64_t(left) * (p + 1) / P);
  }
  __device__ __forceinline__ int count() const { return rounds * mbs + (lu1 - lu0); }
  __device__ __forceinline__ void unit(const GemmArgs& g, int i, int& r, int& nb, int& mb, int& panel) const {
    if (i < rounds * mbs) {
      const int k = i / mbs;
      mb = i - k * mbs;
      panel = k * P + p;
    } else {
      const int j = lu0 + (i - rounds * mbs);
      panel = rounds * P + j / mbs;
      mb = j - (j / mbs) * mbs;
    }
    r = panel / g.tiles_n;
    nb = panel - r * g.tiles_n;
  }
};

template <typename TO>
__global__ void __launch_bounds__(kGemmThreads, 1) gemm_pair_kernel(const __grid_constant__ RankMaps maps, GemmArgs g,
                                                                    uint32_t in_fmt) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int kblocks = g.K / BK;
  const int NS = pair_stages(kblocks);
  uint8_t* bpan = smem;                                // kblocks x 16 KB, B half panel
  uint8_t* aring = bpan + kblocks * kPairBBytes;       // NS x 16 KB
  uint8_t* epi = aring + NS * kPairABytes;             // 1024-aligned staging
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + kPairEpiBytes);  // leader: both A halves of a stage
  uint64_t* empty = full + NS;                         // both: the pair MMAs on a stage retired
  uint64_t* bfull = empty + NS;                        // leader: both B halves of a panel
  uint64_t* bempty = bfull + 1;                        // both: the pair MMAs on a panel retired
  uint64_t* tfull = bempty + 1;                        // [2] both: accumulator ready
  uint64_t* tempty = tfull + 2;                        // [2] leader: both epilogues drained it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  if (warp == 0 && lane == 0) {
    // full / bfull: the LEADER's producer arrives once with the bytes of both
    // CTAs' loads; the peer's loads only complete transactions on it
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(bfull, 1);
    mbar_init(bempty, 1);
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's barriers exist before any remote arrive / multicast commit
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const PairSched ps(g, int(gridDim.x >> 1), int(blockIdx.x >> 1));
  const int nu = ps.count();

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs)
      const uint32_t full_l = mapa_leader(full), bfull_l = mapa_leader(bfull);
      // A row blocks are re-read by the other pairs on the rank: keep them in L2
      // against the C write stream (stores are evict_first)
      const uint64_t keep = createpolicy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      int panel = -1, npanel = 0;
      for (int u = 0; u < nu; ++u) {
        int r, nb, mb, pid;
        ps.unit(g, u, r, nb, mb, pid);
        if (pid != panel) {
          if (npanel > 0) mbar_wait(bempty, uint32_t(npanel - 1) & 1u);  // the old panel's MMAs retired
          if (crank == 0) mbar_expect_tx(bfull, uint32_t(2 * kblocks * kPairBBytes));
          for (int kb = 0; kb < kblocks; ++kb)
#pragma unroll
            for (int j = 0; j < 2; ++j)
              tma_load_2d_pair(bpan + kb * kPairBBytes + j * kMnBlockBytes, &maps.b[r],
                               nb * 256 + int(crank) * 128 + j * 64, kb * BK, bfull_l, keep);
          panel = pid;
          ++npanel;
        }
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (g.diag & 2) {  // profiling only: no A loads (MMAs on stale smem)
            if (crank == 0) mbar_arrive(&full[stage]);
          } else {
            if (crank == 0) mbar_expect_tx(&full[stage], uint32_t(2 * kPairABytes));
            tma_load_2d_pair(aring + stage * kPairABytes, &maps.a[r], kb * BK, mb * 256 + int(crank) * BM,
                             full_l + uint32_t(stage * 8), keep);
          }
          if (++stage == NS) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && crank == 0) {  // ---- MMA issuer (leader)
      const uint32_t idesc = make_idesc_pair(in_fmt);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int panel = -1, npanel = 0;
      for (int u = 0; u < nu; ++u) {
        int r, nb, mb, pid;
        ps.unit(g, u, r, nb, mb, pid);
        if (pid != panel) {
          if (npanel > 0) mma_commit_pair(bempty);  // frees the old panel once its MMAs retire
          mbar_wait(bfull, uint32_t(npanel) & 1u);
          tc_fence_after();
          panel = pid;
          ++npanel;
        }
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + uint32_t(acc * kAccStride);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t da = sw128_desc(aring + stage * kPairABytes);
          const uint64_t db = sw128_mn_desc(bpan + kb * kPairBBytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_f16_pair(d, da + 2 * k, db + uint64_t(k) * ((16 * 128) >> 4), idesc, (kb | k) != 0);
          mma_commit_pair(&empty[stage]);
          if (++stage == NS) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_pair(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4 && warp < 8) {  // ---- epilogue (both CTAs): rows mb*256 + crank*128 + ...
    const int q = warp & 3;
    uint8_t* stg = epi + q * kPairEpiBufs * 4096;
    constexpr int kCols = 128 / int(sizeof(TO));
    const uint32_t tempty_l = mapa_leader(tempty);
    const uint64_t stream = createpolicy_evict_first();
    int acc = 0, buf = 0;
    uint32_t acc_phase = 0;
    for (int u = 0; u < nu; ++u) {
      int r, nb, mb, pid;
      ps.unit(g, u, r, nb, mb, pid);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem + (uint32_t(q * 32) << 16) + uint32_t(acc * kAccStride);
#pragma unroll 1
      for (int cc = 0; cc < 256 / kCols; ++cc) {
        // this staging buffer was last read by the store issued kPairEpiBufs chunks ago
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kPairEpiBufs - 1) : "memory");
        __syncwarp();
        uint8_t* row = stg + buf * 4096 + lane * 128;
        uint32_t h[32];
        if constexpr (sizeof(TO) == 4) {
          uint32_t v[32];
          tmem_ld32(tbase + uint32_t(cc * 32), v);
#pragma unroll
          for (int i = 0; i < 32; ++i) h[i] = v[i];
        } else {
          uint32_t v[32], w[32];
          tmem_ld32(tbase + uint32_t(cc * 64), v);
          tmem_ld32(tbase + uint32_t(cc * 64 + 32), w);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            TO lo = from_f32<TO>(__uint_as_float(v[2 * i])), hi = from_f32<TO>(__uint_as_float(v[2 * i + 1]));
            h[i] = uint32_t(*reinterpret_cast<uint16_t*>(&lo)) | (uint32_t(*reinterpret_cast<uint16_t*>(&hi)) << 16);
            TO lo2 = from_f32<TO>(__uint_as_float(w[2 * i])), hi2 = from_f32<TO>(__uint_as_float(w[2 * i + 1]));
            h[16 + i] =
                uint32_t(*reinterpret_cast<uint16_t*>(&lo2)) | (uint32_t(*reinterpret_cast<uint16_t*>(&hi2)) << 16);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint4*>(row + ((j ^ (lane & 7)) << 4)) =
              make_uint4(h[4 * j], h[4 * j + 1], h[4 * j + 2], h[4 * j + 3]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0 && !(g.diag & 1)) {  // diag 1 (profiling only): no C stores
          tma_store_2d_hint(&maps.c[r], stg + buf * 4096, nb * 256 + cc * kCols, mb * 256 + int(crank) * BM + q * 32,
                            stream);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (++buf == kPairEpiBufs) buf = 0;
      }
      // this CTA's 128 epilogue threads are done with the accumulator: one
      // arrive on the leader's barrier (count 2: both CTAs)
      tc_fence_before();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (warp == 4 && lane == 0) mbar_arrive_cl(tempty_l + uint32_t(acc * 8));
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves (or frees TMEM) while the pair's MMAs, commits or loads may touch it
  tc_fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
}

// ---- MP layer as ONE all-gather -> GEMM kernel (mp_overlap.json) ----
// OverlapGroup{MatMul, FusedAllReduce{dropout(layer + b) + r}} computes, for
// the output column block c owned by rank c,
//     out[:, c] = dropout(sum_r A_r x B_r[:, c] + b[c], rate) + r[:, c]
// and gathers it to every rank. The reference forms every rank's partial
// product [rows x cols] and reduce-scatters it (runtime.hpp:471-516). Here the
// partial products never exist: the pair of CTAs that owns (c, 256-row block)
// streams A_r (rows x k_local) and B_r[:, c] of EVERY rank r through one K
// loop of W * k_local (TMA from the peers' memory: the all-gather of the
// activations, overlapped with the MMAs k-block by k-block), accumulates in
// fp32 TMEM, and its epilogue applies bias + dropout + residual and stores the
// finished tile into every rank's `out` (the AllGather push). The same NVLink
// bytes as the RS (every rank's A slice instead of every rank's partial
// block), no partial write-back, no second kernel. FAST math: the sum is
// accumulated in fp32 over the whole K and rounded once to 16 bits in the
// epilogue (the two-kernel schedule rounds every rank's partial product to 16
// bits and folds them in fp32 ring order), masks bit-exact (global flat index
// as the dropout counter, state.hpp:178-181).
// Shapes: per = cols / W a multiple of 128, run as sub-blocks of PER = 384,
// 256 or 128 columns (two pair MMAs per k-step at 384: N = 256 and N = 128),
// rows % 256 == 0, k_local % 64 == 0. 512 threads:
// warp 0 producer, warp 1 MMA issuer (leader), warp 2 TMEM allocator, warps
// 2-15 epilogue (4-11 also drain TMEM). On one GPU the 8 pushes of every
// tile (403 MB at C3) bound it: profiles/r02_mp_ag_gemm.json.
constexpr int kAgStages1 = 3;
constexpr int kAg1Threads = 512;  // warp 0 producer, 1 MMA, 2-15 epilogue (4-11 also drain TMEM)
struct AgMaps {
  CUtensorMap a[kMaxRanks];    // A_r: [rows, k_local], boxes 64 k x 128 rows
  CUtensorMap b[kMaxRanks];    // B_r: [k_local, cols], boxes 64 n x 64 k (MN-major)
  CUtensorMap out[kMaxRanks];  // out of every rank: boxes 64 cols x 128 rows
};
struct AgArgs {
  RankSet rs;  // DISTRIBUTED: entry / exit barrier with the peers whose A, B we read and whose out we write
  const uint16_t* bias[kMaxRanks];  // b (replicated) of each owner computed here
  const uint16_t* res[kMaxRanks];   // r (replicated) of each owner computed here
  int rows, cols, per, k_local, W;
  int n0, n1;
  int owner0, owners;  // column blocks computed by this launch
  int dst;             // destination ranks of the output push (the group)
  float frate_scale;
  uint64_t seed, key, thresh;
  int f16;             // 16-bit type: 1 = fp16, 0 = bf16
  int diag;            // COCONET_GEMM_DIAG (profiling only): 1 = no epilogue math / stores, 2 = no operand loads
};

__device__ __forceinline__ uint32_t make_idesc_pair_n(uint32_t in_fmt, int n) {
  return (1u << 4) | (in_fmt << 7) | (in_fmt << 10) | (1u << 16) | (uint32_t(n >> 3) << 17) |
         (uint32_t(256 >> 4) << 24);
}

__device__ __forceinline__ float h16_to_f32(uint16_t h, int f16) {
  return f16 ? __half2float(__ushort_as_half(h)) : __bfloat162float(__ushort_as_bfloat16(h));
}
__device__ __forceinline__ uint16_t f32_to_h16(float x, int f16) {
  return f16 ? __half_as_ushort(__float2half_rn(x)) : __bfloat16_as_ushort(__float2bfloat16_rn(x));
}

template <int PER>
__global__ void __launch_bounds__(kAg1Threads, 1) mp_ag_gemm_kernel(const __grid_constant__ AgMaps maps, AgArgs g,
                                                                   uint32_t in_fmt) {
  // A unit is (256-row block, owner column block): ONE K loop of W * k_local
  // into a PER-column TMEM accumulator (two MMAs per k-step at PER = 384:
  // N = 256 and N = 128). The epilogue first drains the accumulator into a
  // shared-memory unit buffer (16-bit, one rounding of the fp32 sum) and
  // releases TMEM at once, so the next unit's MMAs overlap the bias +
  // dropout + residual pass over that buffer and its pushes.
  constexpr int kW0 = PER < 256 ? PER : 256, kW1 = PER - kW0;
  constexpr int kStage = kPairABytes + (PER / 2) * 128;  // A 16 KB + this CTA's PER/2 B columns
  constexpr int kChunks = PER / 64;                      // 64-column x 128-row chunks of the unit buffer
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint8_t* ubuf = ring + kAgStages1 * kStage;  // 1024-aligned: kStage is a multiple of 1024
  uint64_t* full = reinterpret_cast<uint64_t*>(ubuf + kChunks * 16384);
  uint64_t* empty = full + kAgStages1;
  uint64_t* tfull = empty + kAgStages1;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kAgStages1; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  edge_barrier(g.rs, 0);  // DISTRIBUTED: every peer's A, B are ready (VIRTUAL: stream order)
  const int mbs = g.rows / 256;
  const int nsub = g.per / PER;  // PER-column sub-blocks of an owner's column block
  const int units = g.owners * mbs * nsub;
  const int P = int(gridDim.x >> 1), pr = int(blockIdx.x >> 1);
  const int kb_per = g.k_local / BK, kb_all = g.W * kb_per;
  // unit u -> (row block, owner, sub-block), row-block-major: the pairs
  // running together read the same A row blocks (every owner needs them)
  auto decode = [&](int u, int& mb, int& c, int& cb) {
    const int per_mb = g.owners * nsub;
    mb = u / per_mb;
    const int rem = u - mb * per_mb;
    c = g.owner0 + rem / nsub;
    cb = c * g.per + (rem - (rem / nsub) * nsub) * PER;  // first output column of the unit
  };
  if (warp == 0) {
    if (lane == 0) {  // ---- producer (both CTAs)
      const uint32_t full_l = mapa_leader(full);
      const uint64_t keep = createpolicy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pr; u < units; u += P) {
        int mb, c, cb;
        decode(u, mb, c, cb);
        for (int kk = 0; kk < kb_all; ++kk) {
          const int r = kk / kb_per, kb = kk - r * kb_per;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = ring + stage * kStage;
          if (g.diag & 2) {
            if (crank == 0) mbar_arrive(&full[stage]);
          } else {
            if (crank == 0) mbar_expect_tx(&full[stage], uint32_t(2 * kStage));
            const uint32_t fb = full_l + uint32_t(stage * 8);
            tma_load_2d_pair(st, &maps.a[r], kb * BK, mb * 256 + int(crank) * BM, fb, keep);
            uint8_t* sb = st + kPairABytes;
            for (int j = 0; j < kW0 / 128; ++j)  // part 0: this CTA's kW0/2 columns
              tma_load_2d_pair(sb + j * kMnBlockBytes, &maps.b[r], cb + int(crank) * (kW0 / 2) + j * 64, kb * BK,
                               fb, keep);
            sb += (kW0 / 128) * kMnBlockBytes;
            for (int j = 0; j < kW1 / 128; ++j)  // part 1: this CTA's kW1/2 columns
              tma_load_2d_pair(sb + j * kMnBlockBytes, &maps.b[r], cb + kW0 + int(crank) * (kW1 / 2) + j * 64,
                               kb * BK, fb, keep);
          }
          if (++stage == kAgStages1) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && crank == 0) {  // ---- MMA issuer (leader)
      const uint32_t id0 = make_idesc_pair_n(in_fmt, kW0), id1 = make_idesc_pair_n(in_fmt, kW1 > 0 ? kW1 : 128);
      int stage = 0;
      uint32_t phase = 0, tph = 0;
      for (int u = pr; u < units; u += P) {
        mbar_wait(tempty, tph ^ 1);  // both CTAs drained the accumulator
        tc_fence_after();
        for (int kk = 0; kk < kb_all; ++kk) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          uint8_t* st = ring + stage * kStage;
          const uint64_t da = sw128_desc(st);
          const uint64_t d0 = sw128_mn_desc(st + kPairABytes);
          const uint64_t d1 = sw128_mn_desc(st + kPairABytes + (kW0 / 128) * kMnBlockBytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            mma_f16_pair(tmem, da + 2 * k, d0 + uint64_t(k) * ((16 * 128) >> 4), id0, (kk | k) != 0);
            if constexpr (kW1 > 0)
              mma_f16_pair(tmem + uint32_t(kW0), da + 2 * k, d1 + uint64_t(k) * ((16 * 128) >> 4), id1,
                           (kk | k) != 0);
          }
          mma_commit_pair(&empty[stage]);
          if (++stage == kAgStages1) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_pair(tfull);
        tph ^= 1;
      }
    }
  } else {  // ---- epilogue (both CTAs): warps 2-15
    // Warps 4-11 drain the accumulator (TMEM lane quarter q = warp % 4,
    // column half h) into the shared-memory unit buffer as 16-bit values and
    // release TMEM; then all 14 warps run bias + dropout + residual over the
    // buffer, thread t taking 32-column groups (t % 12 of a 384-wide row), so
    // the residual loads are coalesced; one thread pushes the unit to every
    // rank's `out`.
    constexpr int kEpiThreads = kAg1Threads - 64;  // warps 2..15
    constexpr int kGroups = PER / 32;              // 32-column groups per row
    const int et = int(threadIdx.x) - 64;
    const bool pusher = et == 0;
    const bool drainer = warp >= 4 && warp < 12;
    const int q = warp & 3, h = (warp - 4) >> 2;
    const uint32_t tempty_l = mapa_leader(tempty);
    const uint64_t stream = createpolicy_evict_first();
    constexpr int kHalf = PER / 2;
    uint32_t tph = 0;
    for (int u = pr; u < units; u += P) {
      int mb, c, cb;
      decode(u, mb, c, cb);
      const int oi = c - g.owner0;
      const int row0 = mb * 256 + int(crank) * BM;
      // the unit buffer is free once the previous unit's pushes have read it
      if (pusher) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
      if (drainer) {
        mbar_wait(tfull, tph);
        tc_fence_after();
        const int lrow = q * 32 + lane;
        const uint32_t tbase = tmem + (uint32_t(q * 32) << 16) + uint32_t(h * kHalf);
#pragma unroll 1
        for (int s32 = 0; s32 < kHalf / 32; ++s32) {
          uint32_t v[32];
          tmem_ld32(tbase + uint32_t(s32 * 32), v);
          const int col = h * kHalf + s32 * 32;  // column inside the unit
          uint8_t* rowp = ubuf + (col / 64) * 16384 + lrow * 128;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t w4[4];
#pragma unroll
            for (int t = 0; t < 4; ++t)
              w4[t] = uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(__uint_as_float(v[8 * j + 2 * t])))) |
                      (uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(__uint_as_float(v[8 * j + 2 * t + 1]))))
                       << 16);
            *reinterpret_cast<uint4*>(rowp + (((((col % 64) / 8) + j) ^ (lane & 7)) << 4)) =
                make_uint4(w4[0], w4[1], w4[2], w4[3]);
          }
        }
        tc_fence_before();
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
      if (warp == 4 && lane == 0) mbar_arrive_cl(tempty_l);  // both CTAs' arrivals release the accumulator
      // bias + dropout + residual over the buffer, in place
      if (!(g.diag & 1)) {
#pragma unroll 1
        for (int it = et; it < BM * kGroups; it += kEpiThreads) {
          const int lrow = it / kGroups, grp = it - lrow * kGroups;
          const int col = grp * 32, gcol = cb + col, row = row0 + lrow;
          uint8_t* rowp = ubuf + (col / 64) * 16384 + lrow * 128;
          const uint4* rp = reinterpret_cast<const uint4*>(g.res[oi] + int64_t(row) * g.cols + gcol);
          const uint4* bp = reinterpret_cast<const uint4*>(g.bias[oi] + gcol);
          uint4 rr[4], bb[4], aa[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            rr[j] = __ldg(rp + j);
            bb[j] = __ldg(bp + j);
            aa[j] = *reinterpret_cast<const uint4*>(rowp + (((((col % 64) / 8) + j) ^ (lrow & 7)) << 4));
          }
          const uint16_t* r16 = reinterpret_cast<const uint16_t*>(rr);
          const uint16_t* b16 = reinterpret_cast<const uint16_t*>(bb);
          const uint16_t* a16 = reinterpret_cast<const uint16_t*>(aa);
          uint32_t o[16];
          const uint64_t gi0 = uint64_t(row) * uint64_t(g.cols) + uint64_t(gcol);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float y[2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              const int j = 2 * i + t;
              const float x = __bfloat162float(__ushort_as_bfloat16(a16[j])) + h16_to_f32(b16[j], g.f16);
              const bool kp = dropout_keep_bits(g.seed, g.key, gi0 + uint64_t(j), g.thresh);
              y[t] = (kp ? x * g.frate_scale : 0.0f) + h16_to_f32(r16[j], g.f16);
            }
            o[i] = uint32_t(f32_to_h16(y[0], g.f16)) | (uint32_t(f32_to_h16(y[1], g.f16)) << 16);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint4*>(rowp + (((((col % 64) / 8) + j) ^ (lrow & 7)) << 4)) =
                make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
        }
      }
      // the AllGather push: the finished unit into every rank's out
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
      if (pusher) {
        if (!(g.diag & 1))
          for (int dd = 0; dd < ((g.diag & 8) ? 1 : g.dst); ++dd)  // diag 8 (profiling only): one destination
            for (int j = 0; j < kChunks; ++j)
              tma_store_2d_hint(&maps.out[dd], ubuf + j * 16384, cb + j * 64, row0, stream);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      tph ^= 1;
    }
    if (pusher) {
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async.global;" ::: "memory");  // the pushes before the exit barrier's release
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  edge_barrier(g.rs, 1);  // DISTRIBUTED: our pushes into every peer's out have landed
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
}

template <int PER>
constexpr int ag_smem() {
  return kAgStages1 * (kPairABytes + (PER / 2) * 128) + (PER / 64) * 16384 + 1024 + 512;
}



// EXACT: C = A x B with fp64 accumulation in k order (eval_matmul).
struct ExactArgs {
  const float* a[kMaxRanks];
  const float* b[kMaxRanks];
  float* c[kMaxRanks];
  int M, N, K;
};

__global__ void __launch_bounds__(256) gemm_exact_kernel(ExactArgs g) {
  __shared__ float As[64][33];
  __shared__ float Bs[32][65];
  const int r = blockIdx.z;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < g.K; k0 += 32) {
    for (int i = threadIdx.x; i < 64 * 32; i += 256) {
      const int mm = i / 32, kk = i % 32;
      As[mm][kk] = (m0 + mm < g.M && k0 + kk < g.K) ? g.a[r][int64_t(m0 + mm) * g.K + k0 + kk] : 0.f;
      const int kb = i / 64, nb = i % 64;
      Bs[kb][nb] = (k0 + kb < g.K && n0 + nb < g.N) ? g.b[r][int64_t(k0 + kb) * g.N + n0 + nb] : 0.f;
    }
    __syncthreads();
    const int kmax = min(32, g.K - k0);
    for (int kk = 0; kk < kmax; ++kk) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          acc[i][j] = __fma_rn(double(As[ty * 4 + i][kk]), double(Bs[kk][tx * 4 + j]), acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < g.M && n < g.N) g.c[r][int64_t(m) * g.N + n] = float(acc[i][j]);
    }
}

// ---- host side ---------------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_map(CUtensorMap* map, const void* base, int elem, uint64_t inner, uint64_t outer, uint32_t box_inner,
             uint32_t box_outer) {
  auto fn = encode_fn();
  if (!fn) return set_error(COCONET_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const uint64_t esz = elem == COCONET_F32 ? 4 : 2;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * esz};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = elem == COCONET_BF16  ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                 : elem == COCONET_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                       : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUresult r = fn(map, dt, 2,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(COCONET_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return COCONET_OK;
}

struct TcPlan {
  RankMaps maps;
  GemmArgs g;
  int bn;
};

// Prepares the tcgen05 launch for every local rank of `group`: encodes the
// TMA maps (A K-major, B read MN-major in place, C).
int plan_tc(coconet_ctx* c, int group, const void* a, const void* b, void* cc, int in_elem, int out_elem, int64_t m,
            int64_t n, int64_t k, cudaStream_t s, TcPlan* p) {
  if (m % BM) return set_error(COCONET_ERR_UNSUPPORTED, "M must be a multiple of 128");
  if (k % BK) return set_error(COCONET_ERR_UNSUPPORTED, "K must be a multiple of 64");
  int bn = n % 256 == 0 ? 256 : (n % 192 == 0 ? 192 : (n % 128 == 0 ? 128 : 0));
  if (!bn) return set_error(COCONET_ERR_UNSUPPORTED, "N must be a multiple of 128 or 192");
  int64_t ao = 0, bo = 0, co = 0;
  int rc = heap_offset(c, a, &ao);
  if (!rc) rc = heap_offset(c, b, &bo);
  if (!rc) rc = heap_offset(c, cc, &co);
  if (rc) return rc;
  const coconet_group_s& grp = c->groups[size_t(group)];
  const int nl = local_ranks(c, group);
  std::memset(&p->maps, 0, sizeof(p->maps));
  std::memset(&p->g, 0, sizeof(p->g));
  for (int i = 0; i < nl; ++i) {
    const int wr = c->mode == COCONET_MODE_VIRTUAL ? grp.first + i : c->rank;
    char* heap = c->heap[wr];
    rc = make_map(&p->maps.a[i], heap + ao, in_elem, uint64_t(k), uint64_t(m), BK, BM);
    if (!rc) rc = make_map(&p->maps.a_half[i], heap + ao, in_elem, uint64_t(k), uint64_t(m), BK, BM / 2);
    // B in its natural row-major [K, N] layout, read MN-major (64 n x 64 k boxes)
    if (!rc) rc = make_map(&p->maps.b[i], heap + bo, in_elem, uint64_t(n), uint64_t(k), 64, BK);
    if (!rc)
      rc = make_map(&p->maps.c[i], heap + co, out_elem, uint64_t(n), uint64_t(m), out_elem == COCONET_F32 ? 32 : 64, 32);
    if (rc) return rc;
    p->g.c[i] = heap + co;
  }
  CN_CUDA(cudaGetLastError());
  p->g.M = int(m);
  p->g.N = int(n);
  p->g.K = int(k);
  p->g.ranks = nl;
  static const int diag = getenv("COCONET_GEMM_DIAG") ? atoi(getenv("COCONET_GEMM_DIAG")) : 0;
  p->g.diag = diag;
  p->g.tiles_m = int(m / BM);
  p->g.tiles_n = int(n / bn);
  p->bn = bn;
  return COCONET_OK;
}

template <int BN, typename TO, bool FUSED>
int launch_tc_t(coconet_ctx* c, TcPlan* p, uint32_t in_fmt, const OvArgs* ov, cudaStream_t s) {
  const int smem = Cfg<BN>::SMEM;
  const int total = p->g.ranks * p->g.tiles_m * p->g.tiles_n;
  OvArgs none{};
  const OvArgs& o = ov ? *ov : none;
  if constexpr (!FUSED) {
    // BN = 256 with a B half panel that fits: the 2-SM pair kernel (B resident;
    // COCONET_GEMM_PAIR=0 disables it)
    const char* pe = getenv("COCONET_GEMM_PAIR");
    if (BN == 256 && !(pe && pe[0] == '0') && p->g.tiles_m % 2 == 0 && p->g.K <= kPairKMax) {
      const int psmem = pair_smem(p->g.K / BK);
      auto fn = gemm_pair_kernel<TO>;
      CN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, psmem));
      const int units = p->g.ranks * p->g.tiles_n * (p->g.tiles_m / 2);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(unsigned(2 * std::min(units, c->sm_count / 2)));
      cfg.blockDim = dim3(kGemmThreads);
      cfg.dynamicSmemBytes = size_t(psmem);
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      CN_CUDA(cudaLaunchKernelEx(&cfg, fn, p->maps, p->g, in_fmt));
      c->launches++;
      return COCONET_OK;
    }
    // COCONET_GEMM_MC: 0 = no clusters, a = pairs share A (default), b = pairs
    // share B (less L2 -> SM traffic, but no faster end to end at C3's shape:
    // profiles/r01_gemm_diag.json)
    const char* e = getenv("COCONET_GEMM_MC");
    const char want = e ? e[0] : 'a';
    const bool mc_b = (want == 'b') && p->g.tiles_m % 2 == 0 && (BN / 64) % 2 == 0;
    const bool mc_a = !mc_b && want != '0' && p->g.tiles_n % 2 == 0;
    if (mc_a || mc_b) {  // 2-CTA clusters sharing an operand by multicast
      auto fn = mc_b ? gemm_tc_kernel<BN, TO, false, 2> : gemm_tc_kernel<BN, TO, false, 1>;
      CN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(unsigned(2 * std::min(total / 2, c->sm_count / 2)));
      cfg.blockDim = dim3(kGemmThreads);
      cfg.dynamicSmemBytes = size_t(smem);
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      CN_CUDA(cudaLaunchKernelEx(&cfg, fn, p->maps, p->g, in_fmt, o));
    } else {
      auto fn = gemm_tc_kernel<BN, TO, false, 0>;
      CN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      const int grid = std::min(total, c->sm_count);
      fn<<<grid, kGemmThreads, smem, s>>>(p->maps, p->g, in_fmt, o);
      CN_CUDA(cudaGetLastError());
    }
  } else {
    // every CTA both computes tiles and all-reduces: co-residency (one CTA
    // per SM) is guaranteed by the cooperative launch, so comm warps spinning
    // on tile flags can never starve the CTAs that publish them
    auto fn = gemm_tc_kernel<BN, TO, true, 0>;
    CN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int grid = c->sm_count;
    void* args[] = {const_cast<RankMaps*>(&p->maps), &p->g, &in_fmt, const_cast<OvArgs*>(&o)};
    CN_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), dim3(grid), dim3(kFusedThreads), args, smem, s));
  }
  c->launches++;
  return COCONET_OK;
}

template <bool FUSED>
int launch_tc(coconet_ctx* c, TcPlan* p, int in_elem, int out_elem, const OvArgs* ov, cudaStream_t s) {
  const uint32_t fmt = in_elem == COCONET_BF16 ? 1u : 0u;
  const bool f32 = out_elem == COCONET_F32;
  const bool bf = out_elem == COCONET_BF16;
  if (FUSED && f32) return set_error(COCONET_ERR_UNSUPPORTED, "the fused overlap keeps 16-bit partials");
  switch (p->bn) {
    case 256: return f32 ? launch_tc_t<256, float, false>(c, p, fmt, ov, s)
                         : (bf ? launch_tc_t<256, __nv_bfloat16, FUSED>(c, p, fmt, ov, s)
                               : launch_tc_t<256, __half, FUSED>(c, p, fmt, ov, s));
    case 192: return f32 ? launch_tc_t<192, float, false>(c, p, fmt, ov, s)
                         : (bf ? launch_tc_t<192, __nv_bfloat16, FUSED>(c, p, fmt, ov, s)
                               : launch_tc_t<192, __half, FUSED>(c, p, fmt, ov, s));
    default: return f32 ? launch_tc_t<128, float, false>(c, p, fmt, ov, s)
                        : (bf ? launch_tc_t<128, __nv_bfloat16, FUSED>(c, p, fmt, ov, s)
                              : launch_tc_t<128, __half, FUSED>(c, p, fmt, ov, s));
  }
}

// The all-gather -> GEMM schedule of OverlapGroup{MatMul, FusedAllReduce}
// (mp_ag_gemm_kernel). Returns COCONET_ERR_UNSUPPORTED for shapes it does not
// take (the caller falls back to the two-kernel schedule).
int launch_ag_gemm(coconet_ctx* c, int group, const void* a, const void* w, const void* b, const void* r, void* out,
                   int in_elem, int64_t rows, int64_t cols, int64_t k_local, const coconet_bdr_params* hp,
                   cudaStream_t s) {
  const int W = c->groups[size_t(group)].size;
  const int64_t per = cols / W;
  // sub-block width: 384, 256 or 128 columns (the TMEM accumulator)
  const int sbw = per % 384 == 0 ? 384 : per % 256 == 0 ? 256 : per % 128 == 0 ? 128 : 0;
  if (!sbw || rows % 256 || k_local % BK || rows > INT32_MAX ||
      int64_t(rows) * cols > (int64_t(1) << 40) || W > kMaxRanks)
    return COCONET_ERR_UNSUPPORTED;
  int64_t ao = 0, wo = 0, bo = 0, ro = 0, oo = 0;
  int rc = heap_offset(c, a, &ao);
  if (!rc) rc = heap_offset(c, w, &wo);
  if (!rc) rc = heap_offset(c, b, &bo);
  if (!rc) rc = heap_offset(c, r, &ro);
  if (!rc) rc = heap_offset(c, out, &oo);
  if (rc) return rc;
  if ((ao | wo | bo | ro | oo) % 16) return COCONET_ERR_UNSUPPORTED;
  AgMaps maps;  // the kernel parameter (3 KB of tensor maps), copied at launch
  AgArgs g{};
  rc = make_rankset(c, group, &g.rs);
  if (rc) return rc;
  const coconet_group_s& grp = c->groups[size_t(group)];
  for (int q = 0; q < W; ++q) {
    char* heap = c->heap[grp.first + q];  // VIRTUAL: this device; DISTRIBUTED: the peer mapping
    rc = make_map(&maps.a[q], heap + ao, in_elem, uint64_t(k_local), uint64_t(rows), BK, BM);
    if (!rc) rc = make_map(&maps.b[q], heap + wo, in_elem, uint64_t(cols), uint64_t(k_local), 64, BK);
    if (!rc) rc = make_map(&maps.out[q], heap + oo, in_elem, uint64_t(cols), uint64_t(rows), 64, 128);
    if (rc) return rc;
  }
  // owners computed here: every column block (VIRTUAL) or this rank's (DISTRIBUTED)
  g.owner0 = c->mode == COCONET_MODE_VIRTUAL ? 0 : c->rank - grp.first;
  g.owners = c->mode == COCONET_MODE_VIRTUAL ? W : 1;
  for (int i = 0; i < g.owners; ++i) {
    char* heap = c->heap[grp.first + g.owner0 + i];
    g.bias[i] = reinterpret_cast<const uint16_t*>(heap + bo);
    g.res[i] = reinterpret_cast<const uint16_t*>(heap + ro);
  }
  g.rows = int(rows);
  g.cols = int(cols);
  g.per = int(per);
  g.k_local = int(k_local);
  g.W = W;
  g.n0 = std::min(sbw, 256);
  g.n1 = sbw - g.n0;
  g.dst = W;
  g.frate_scale = float(1.0 / (1.0 - hp->rate));
  g.seed = hp->seed;
  g.key = hp->key;
  const double th = std::ceil(hp->rate * 9007199254740992.0);
  g.thresh = th <= 0 ? 0 : (th >= 9007199254740992.0 ? (uint64_t(1) << 53) : uint64_t(th));
  g.f16 = in_elem == COCONET_F16 ? 1 : 0;
  g.diag = getenv("COCONET_GEMM_DIAG") ? atoi(getenv("COCONET_GEMM_DIAG")) : 0;
  const uint32_t fmt = in_elem == COCONET_BF16 ? 1u : 0u;
  const int smem = sbw == 384 ? ag_smem<384>() : sbw == 256 ? ag_smem<256>() : ag_smem<128>();
  auto fn = sbw == 384 ? mp_ag_gemm_kernel<384> : sbw == 256 ? mp_ag_gemm_kernel<256> : mp_ag_gemm_kernel<128>;
  CN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int units = g.owners * int(rows / 256) * int(per / sbw);
  cudaLaunchConfig_t cfg{};
  // DISTRIBUTED: the same grid on every rank (the edge barriers pair CTA b with CTA b)
  cfg.gridDim = dim3(unsigned(2 * (c->mode == COCONET_MODE_VIRTUAL ? std::min(units, c->sm_count / 2)
                                                                    : c->sm_count / 2)));
  cfg.blockDim = dim3(kAg1Threads);
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CN_CUDA(cudaLaunchKernelEx(&cfg, fn, maps, g, fmt));
  c->launches++;
  return COCONET_OK;
}

constexpr size_t kTileFlagBytes = kCountersOff - kTileFlagsOff;  // per group: up to 16384 tiles

}  // namespace

extern "C" {

int coconet_matmul(coconet_ctx_t c, int group, const void* a, const void* b, void* cc, int in_elem, int out_elem,
                   int64_t m, int64_t n, int64_t k, int math, void* stream) {
  if (!c || !a || !b || !cc) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  if (!valid_group(c, group)) return set_error(COCONET_ERR_NO_SUCH_RANK, "no such group");
  if (m <= 0 || n <= 0 || k <= 0 || m > INT32_MAX || n > INT32_MAX || k > INT32_MAX)
    return set_error(COCONET_ERR_SHAPE_MISMATCH, "bad matmul shape");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (math == COCONET_MATH_EXACT) {
    if (in_elem != COCONET_F32 || out_elem != COCONET_F32)
      return set_error(COCONET_ERR_UNSUPPORTED, "EXACT matmul takes f32 inputs and output");
    int64_t ao = 0, bo = 0, co = 0;
    int rc = heap_offset(c, a, &ao);
    if (!rc) rc = heap_offset(c, b, &bo);
    if (!rc) rc = heap_offset(c, cc, &co);
    if (rc) return rc;
    ExactArgs g{};
    const coconet_group_s& grp = c->groups[size_t(group)];
    const int nl = local_ranks(c, group);
    for (int i = 0; i < nl; ++i) {
      char* heap = c->heap[c->mode == COCONET_MODE_VIRTUAL ? grp.first + i : c->rank];
      g.a[i] = reinterpret_cast<const float*>(heap + ao);
      g.b[i] = reinterpret_cast<const float*>(heap + bo);
      g.c[i] = reinterpret_cast<float*>(heap + co);
    }
    g.M = int(m);
    g.N = int(n);
    g.K = int(k);
    dim3 grid(unsigned((n + 63) / 64), unsigned((m + 63) / 64), unsigned(nl));
    gemm_exact_kernel<<<grid, 256, 0, s>>>(g);
    CN_CUDA(cudaGetLastError());
    c->launches++;
    return COCONET_OK;
  }
  if (in_elem != COCONET_BF16 && in_elem != COCONET_F16)
    return set_error(COCONET_ERR_UNSUPPORTED, "FAST matmul runs on tcgen05 with bf16/f16 inputs");
  TcPlan p;
  int rc = plan_tc(c, group, a, b, cc, in_elem, out_elem, m, n, k, s, &p);
  if (rc) return rc;
  return launch_tc<false>(c, &p, in_elem, out_elem, nullptr, s);
}

int coconet_mm_overlap_fused_ar(coconet_ctx_t c, int group, const void* a, const void* w, const void* b,
                                const void* r, void* partial, void* out, int in_elem, int64_t rows, int64_t cols,
                                int64_t k_local, const coconet_bdr_params* hp, void* stream) {
  if (!c || !hp) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  if (!valid_group(c, group)) return set_error(COCONET_ERR_NO_SUCH_RANK, "no such group");
  if (in_elem != COCONET_BF16 && in_elem != COCONET_F16)
    return set_error(COCONET_ERR_UNSUPPORTED, "the overlapped MatMul runs on tcgen05 (bf16/f16)");
  const int W = c->groups[size_t(group)].size;
  if (cols % W) return set_error(COCONET_ERR_DIVISIBILITY, "column extent does not divide over the group");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // Schedule: on one GPU the one-kernel overlap measures slower than GEMM
  // then the fused all-reduce (both halves contend for the same HBM and SM
  // memory pipe), and it has not been measured over NVLink
  // yet, so AUTO runs the two kernels back to back (bitwise the same result)
  // in both modes. COCONET_MP_OVERLAP=fused|sequential forces either.
  // AUTO: the all-gather -> GEMM kernel (no partial products; C3 on one GPU
  // 277 -> see DESIGN.md) when the shape fits, else the two kernels.
  const char* ov_env = getenv("COCONET_MP_OVERLAP");
  const bool want_ag = !ov_env || std::strcmp(ov_env, "aggemm") == 0;
  if (want_ag && W > 1) {
    const int rc = launch_ag_gemm(c, group, a, w, b, r, out, in_elem, rows, cols, k_local, hp, s);
    if (rc != COCONET_ERR_UNSUPPORTED) return rc;
    if (ov_env) return set_error(COCONET_ERR_UNSUPPORTED, "the all-gather -> GEMM schedule does not take this shape");
  }
  const bool sequential = ov_env ? std::strcmp(ov_env, "fused") != 0 : W > 1;
  if (sequential) {
    int rc = coconet_matmul(c, group, a, w, partial, in_elem, in_elem, rows, cols, k_local, COCONET_MATH_FAST, stream);
    if (rc) return rc;
    return coconet_fused_rs_bdr_ag(c, group, partial, b, r, out, in_elem, rows, cols, hp, stream);
  }
  TcPlan p;
  int rc = plan_tc(c, group, a, w, partial, in_elem, in_elem, rows, cols, k_local, s, &p);
  if (rc) return rc;
  if (size_t(p.g.tiles_m) * p.g.tiles_n * 4 > kTileFlagBytes)
    return set_error(COCONET_ERR_UNSUPPORTED, "too many tiles for the flag area");
  OvArgs o{};
  rc = make_rankset(c, group, &o.rs);
  if (rc) return rc;
  rc = heap_offset(c, partial, &o.part_off);
  if (!rc) rc = heap_offset(c, b, &o.b_off);
  if (!rc) rc = heap_offset(c, r, &o.r_off);
  if (!rc) rc = heap_offset(c, out, &o.out_off);
  if (rc) return rc;
  if ((o.part_off | o.b_off | o.r_off | o.out_off) % 16 || (cols / W) % 8 || cols % 8)
    return set_error(COCONET_ERR_INVALID_INPUT, "operands, rows and column blocks must be 16-byte aligned");
  // tile flags, arrival counter and unit ticket live in every rank's reserved
  // per-group area (common.cuh)
  o.flag_off = int64_t(group_area(group) + kTileFlagsOff);
  o.cnt_off = int64_t(group_area(group) + kCountersOff);
  o.ticket_off = o.cnt_off + 64;
  o.rows = int(rows);
  o.cols = int(cols);
  o.per = int(cols / W);
  o.tiles_m = p.g.tiles_m;
  o.tiles_n = p.g.tiles_n;
  o.bn = p.bn;
  o.nl = local_ranks(c, group);
  o.n_units = p.g.tiles_m * o.nl * 4;
  o.inv_keep = 1.0 - hp->rate;
  o.frate_scale = float(1.0 / (1.0 - hp->rate));
  o.seed = hp->seed;
  o.key = hp->key;
  double th = std::ceil(hp->rate * 9007199254740992.0);
  o.thresh = th <= 0 ? 0 : uint64_t(th);
  o.math = hp->math;
  // every owner's units each add one arrival to every rank's counter
  const uint32_t arrivals = c->mp_arrivals[group] + uint32_t(p.g.tiles_m) * 4u * uint32_t(W);
  o.arrive_target = arrivals;
  // tickets drawn this call: one per unit, plus the one failing draw with
  // which each of the grid's warps (sm_count CTAs - launch_tc's cooperative
  // grid - x kFusedWarps) leaves the loop
  o.ticket_base = c->mp_tickets[group];
  const uint32_t tickets = o.ticket_base + uint32_t(o.n_units) + uint32_t(c->sm_count) * uint32_t(kFusedWarps);
  for (int i = 0; i < p.g.ranks; ++i)
    p.g.flags[i] = reinterpret_cast<uint32_t*>(p.g.c[i] - o.part_off + o.flag_off);
  p.g.epoch = o.rs.epoch;
  p.g.local_peers = c->mode == COCONET_MODE_VIRTUAL ? 1 : 0;
  rc = launch_tc<true>(c, &p, in_elem, in_elem, &o, s);
  // the host mirrors of the device counters advance only with a launch that
  // happened, so a failed launch cannot leave them ahead of the device
  if (rc == COCONET_OK) {
    c->mp_arrivals[group] = arrivals;
    c->mp_tickets[group] = tickets;
  }
  return rc;
}

}  // extern "C"
