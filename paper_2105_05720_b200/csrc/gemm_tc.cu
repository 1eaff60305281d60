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
//  * Overlap: the RS -> bias+dropout+residual -> AG kernel runs concurrently
//    on a second stream, one work unit per (128-row tile, column block); a unit
//    starts as soon as every rank has published the tiles it covers, so the
//    all-reduce of row tile i overlaps the GEMM of row tiles > i.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>

#include "internal.h"

using namespace coconet;

namespace {

constexpr int BM = 128, BK = 64, STAGES = 4;
constexpr int kGemmThreads = 256;
constexpr int kAccStride = 256;   // TMEM columns per accumulator buffer
constexpr int kTmemCols = 512;

template <int BN> struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

struct RankMaps {
  CUtensorMap a[kMaxRanks];
  CUtensorMap b[kMaxRanks];
};

struct GemmArgs {
  char* c[kMaxRanks];          // C (row-major [M, N]) of each rank computed here
  uint32_t* flags[kMaxRanks];  // per-tile flags of each rank (nullable)
  int M, N, K;
  int ranks;                   // ranks computed by this launch
  int tiles_m, tiles_n;
  uint32_t epoch;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Watchdog: a pipeline that never completes traps (the launch fails with an
// error) instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const unsigned long long t0 = globaltimer();
  while (!mbar_try(bar, parity))
    if (globaltimer() - t0 > 10000000000ull) __trap();
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
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
// both K-major, M = 128, N = BN
template <int BN>
__device__ __forceinline__ uint32_t make_idesc(uint32_t in_fmt) {
  return (1u << 4) | (in_fmt << 7) | (in_fmt << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
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

template <int BN, typename TO>
__global__ void __launch_bounds__(kGemmThreads, 1) gemm_tc_kernel(const __grid_constant__ RankMaps maps, GemmArgs g,
                                                                  uint32_t in_fmt) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg<BN>::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
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
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int total = g.ranks * g.tiles_m * g.tiles_n;
  const int kblocks = g.K / BK;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int r, mt, nt;
        decode_tile(g, t, r, mt, nt);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg<BN>::STAGE_BYTES;
          mbar_expect_tx(&full[stage], Cfg<BN>::STAGE_BYTES);
          tma_load_2d(sa, &maps.a[r], kb * BK, mt * BM, &full[stage]);
          tma_load_2d(sa + Cfg<BN>::A_BYTES, &maps.b[r], kb * BK, nt * BN, &full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer (single thread)
      const uint32_t idesc = make_idesc<BN>(in_fmt);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + uint32_t(acc * kAccStride);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint8_t* sa = smem + stage * Cfg<BN>::STAGE_BYTES;
          const uint64_t da = sw128_desc(sa), db = sw128_desc(sa + Cfg<BN>::A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)  // +32 bytes along K per UMMA_K = 16
            mma_f16(d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          mma_commit(&empty[stage]);  // frees the smem stage once these MMAs retire
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[acc]);  // accumulator complete -> epilogue
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {  // ---- epilogue: TMEM -> registers -> global (+ tile flag)
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int r, mt, nt;
      decode_tile(g, t, r, mt, nt);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = mt * BM + q * 32 + lane;
      TO* crow = reinterpret_cast<TO*>(g.c[r]) + int64_t(row) * g.N + nt * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(acc * kAccStride + c * 32), v);
        store_row32<TO>(crow + c * 32, v);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (g.flags[r] != nullptr) {
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 4 && lane == 0) {
          __threadfence_system();
          st_release_sys(g.flags[r] + mt * g.tiles_n + nt, g.epoch);
        }
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
}

// B [K, N] row-major -> BT [N, K] (K-major operand for the MMA)
template <typename T>
__global__ void transpose_kernel(const T* __restrict__ b, T* __restrict__ bt, int K, int N) {
  __shared__ T tile[32][33];
  const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int k = k0 + i, n = n0 + threadIdx.x;
    if (k < K && n < N) tile[i][threadIdx.x] = b[int64_t(k) * N + n];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int n = n0 + i, k = k0 + threadIdx.x;
    if (k < K && n < N) bt[int64_t(n) * K + k] = tile[threadIdx.x][i];
  }
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
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, elem == COCONET_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(COCONET_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return COCONET_OK;
}

// per-context scratch for transposed weights (grown on demand, never shrunk)
struct Scratch {
  void* p = nullptr;
  size_t bytes = 0;
};
std::mutex g_scratch_mu;
Scratch g_scratch[16];

int scratch_for(coconet_ctx* c, size_t bytes, void** out) {
  std::lock_guard<std::mutex> lk(g_scratch_mu);
  Scratch& s = g_scratch[c->device & 15];
  if (s.bytes < bytes) {
    if (s.p) {
      cudaDeviceSynchronize();
      cudaFree(s.p);
    }
    s.p = nullptr;
    s.bytes = 0;
    CN_CUDA(cudaMalloc(&s.p, bytes));
    s.bytes = bytes;
  }
  *out = s.p;
  return COCONET_OK;
}

struct TcPlan {
  RankMaps maps;
  GemmArgs g;
  int bn;
};

// Prepares the tcgen05 launch for every local rank of `group`: transposes
// each B into scratch and encodes the TMA maps.
int plan_tc(coconet_ctx* c, int group, const void* a, const void* b, void* cc, int in_elem, int64_t m, int64_t n,
            int64_t k, cudaStream_t s, TcPlan* p) {
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
  void* scratch = nullptr;
  rc = scratch_for(c, size_t(nl) * size_t(n * k) * 2, &scratch);
  if (rc) return rc;
  std::memset(&p->maps, 0, sizeof(p->maps));
  std::memset(&p->g, 0, sizeof(p->g));
  for (int i = 0; i < nl; ++i) {
    const int wr = c->mode == COCONET_MODE_VIRTUAL ? grp.first + i : c->rank;
    char* heap = c->heap[wr];
    void* bt = static_cast<char*>(scratch) + size_t(i) * size_t(n * k) * 2;
    dim3 tb(32, 8), tg(unsigned((n + 31) / 32), unsigned((k + 31) / 32));
    transpose_kernel<uint16_t><<<tg, tb, 0, s>>>(reinterpret_cast<const uint16_t*>(heap + bo),
                                                 reinterpret_cast<uint16_t*>(bt), int(k), int(n));
    c->launches++;
    rc = make_map(&p->maps.a[i], heap + ao, in_elem, uint64_t(k), uint64_t(m), BK, BM);
    if (!rc) rc = make_map(&p->maps.b[i], bt, in_elem, uint64_t(k), uint64_t(n), BK, uint32_t(bn));
    if (rc) return rc;
    p->g.c[i] = heap + co;
  }
  CN_CUDA(cudaGetLastError());
  p->g.M = int(m);
  p->g.N = int(n);
  p->g.K = int(k);
  p->g.ranks = nl;
  p->g.tiles_m = int(m / BM);
  p->g.tiles_n = int(n / bn);
  p->bn = bn;
  return COCONET_OK;
}

template <int BN, typename TO>
int launch_tc_t(coconet_ctx* c, TcPlan* p, uint32_t in_fmt, int grid_cap, cudaStream_t s) {
  auto fn = gemm_tc_kernel<BN, TO>;
  const int smem = Cfg<BN>::SMEM;
  CN_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int total = p->g.ranks * p->g.tiles_m * p->g.tiles_n;
  int grid = std::min(total, grid_cap > 0 ? grid_cap : c->sm_count);
  fn<<<grid, kGemmThreads, smem, s>>>(p->maps, p->g, in_fmt);
  CN_CUDA(cudaGetLastError());
  c->launches++;
  return COCONET_OK;
}

int launch_tc(coconet_ctx* c, TcPlan* p, int in_elem, int out_elem, int grid_cap, cudaStream_t s) {
  const uint32_t fmt = in_elem == COCONET_BF16 ? 1u : 0u;
  const bool f32 = out_elem == COCONET_F32;
  const bool bf = out_elem == COCONET_BF16;
  switch (p->bn) {
    case 256: return f32 ? launch_tc_t<256, float>(c, p, fmt, grid_cap, s)
                         : (bf ? launch_tc_t<256, __nv_bfloat16>(c, p, fmt, grid_cap, s)
                               : launch_tc_t<256, __half>(c, p, fmt, grid_cap, s));
    case 192: return f32 ? launch_tc_t<192, float>(c, p, fmt, grid_cap, s)
                         : (bf ? launch_tc_t<192, __nv_bfloat16>(c, p, fmt, grid_cap, s)
                               : launch_tc_t<192, __half>(c, p, fmt, grid_cap, s));
    default: return f32 ? launch_tc_t<128, float>(c, p, fmt, grid_cap, s)
                        : (bf ? launch_tc_t<128, __nv_bfloat16>(c, p, fmt, grid_cap, s)
                              : launch_tc_t<128, __half>(c, p, fmt, grid_cap, s));
  }
}

// ---- the overlap consumer: RS -> bias+dropout+residual -> AG per unit -------

struct OvArgs {
  RankSet rs;            // group ranks (peer heaps)
  int64_t part_off, b_off, r_off, out_off;
  int64_t cnt_off;       // per-rank arrival counter (uint32) in the reserved area
  int64_t flag_off;      // per-rank tile flags
  int rows, cols, per;   // per = cols / W
  int tiles_m, tiles_n, bn;
  uint32_t arrive_target;  // cumulative arrivals expected on this rank's counter
  double inv_keep;
  float frate_scale;
  uint64_t seed, key, thresh;
  int math;
};

__device__ __forceinline__ bool wait_ge(const uint32_t* p, uint32_t want, const RankSet& rs) {
  return wait_flag(p, want, rs);
}

template <typename T>
__global__ void __launch_bounds__(256) overlap_consumer_kernel(OvArgs a) {
  __shared__ char* s_base[kMaxRanks];
  __shared__ int s_ok;
  const RankSet& rs = a.rs;
  if (threadIdx.x < kMaxRanks) s_base[threadIdx.x] = threadIdx.x < rs.world ? rs.base[threadIdx.x] : nullptr;
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  const int W = rs.world, me = rs.rank();
  const int t_lo = (me * a.per) / a.bn, t_hi = ((me + 1) * a.per - 1) / a.bn;  // n-tiles of my block
  const int qpr = a.per / 4;
  for (int mt = blockIdx.x; mt < a.tiles_m; mt += gridDim.x) {
    // wait until every rank published the tiles covering (mt, my column block)
    if (threadIdx.x < W) {
      const uint32_t* fl = reinterpret_cast<const uint32_t*>(s_base[threadIdx.x] + a.flag_off);
      for (int nt = t_lo; nt <= t_hi; ++nt)
        if (!wait_ge(fl + mt * a.tiles_n + nt, rs.epoch, rs)) s_ok = 0;
    }
    __syncthreads();
    if (!s_ok) return;
    for (int i = threadIdx.x; i < 128 * qpr; i += blockDim.x) {
      const int row = mt * 128 + i / qpr;
      const int col = me * a.per + (i % qpr) * 4;
      const int64_t gi = int64_t(row) * a.cols + col;
      float acc[4], x[4];
#pragma unroll
      for (int j = 0; j < kMaxRanks; ++j) {
        if (j >= W) break;
        int src = me + 1 + j;
        src -= src >= W ? W : 0;
        src -= src >= W ? W : 0;
        load4_cg(reinterpret_cast<const T*>(s_base[src] + a.part_off) + gi, x);
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] = j == 0 ? x[e] : __fadd_rn(acc[e], x[e]);
      }
      float b4[4], r4[4], o[4];
      load4(reinterpret_cast<const T*>(s_base[me] + a.b_off) + col, b4);
      load4(reinterpret_cast<const T*>(s_base[me] + a.r_off) + gi, r4);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool keep = dropout_keep_bits(a.seed, a.key, uint64_t(gi + e), a.thresh);
        if (a.math == COCONET_MATH_EXACT) {
          const double sum = __dadd_rn(double(acc[e]), double(b4[e]));
          o[e] = float(__dadd_rn(keep ? __ddiv_rn(sum, a.inv_keep) : 0.0, double(r4[e])));
        } else {
          o[e] = (keep ? (acc[e] + b4[e]) * a.frate_scale : 0.f) + r4[e];
        }
      }
#pragma unroll
      for (int j = 0; j < kMaxRanks; ++j) {
        if (j >= W) break;
        store4(reinterpret_cast<T*>(s_base[j] + a.out_off) + gi, o);
      }
    }
    __syncthreads();
    if (threadIdx.x < W) {  // one arrival per (unit, destination rank)
      __threadfence_system();
      atomicAdd_system(reinterpret_cast<unsigned int*>(s_base[threadIdx.x] + a.cnt_off), 1u);
    }
  }
  // the caller's `out` is complete once every unit of every owner arrived here
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const uint32_t* cnt = reinterpret_cast<const uint32_t*>(s_base[me] + a.cnt_off);
    wait_flag(cnt, a.arrive_target, rs);
  }
}

constexpr size_t kTileFlagBytes = kCountersOff - kTileFlagsOff;  // per group: up to 16384 tiles

std::mutex g_mp_mu;

cudaStream_t g_side[16] = {};
cudaEvent_t g_ev[16][2] = {};

int side_stream(int device, cudaStream_t* s, cudaEvent_t* e0, cudaEvent_t* e1) {
  std::lock_guard<std::mutex> lk(g_mp_mu);
  int d = device & 15;
  if (!g_side[d]) {
    CN_CUDA(cudaStreamCreateWithFlags(&g_side[d], cudaStreamNonBlocking));
    CN_CUDA(cudaEventCreateWithFlags(&g_ev[d][0], cudaEventDisableTiming));
    CN_CUDA(cudaEventCreateWithFlags(&g_ev[d][1], cudaEventDisableTiming));
  }
  *s = g_side[d];
  *e0 = g_ev[d][0];
  *e1 = g_ev[d][1];
  return COCONET_OK;
}

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
  int rc = plan_tc(c, group, a, b, cc, in_elem, m, n, k, s, &p);
  if (rc) return rc;
  return launch_tc(c, &p, in_elem, out_elem, 0, s);
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
  if ((cols / W) % 4) return set_error(COCONET_ERR_UNSUPPORTED, "column block must be a multiple of 4");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  TcPlan p;
  int rc = plan_tc(c, group, a, w, partial, in_elem, rows, cols, k_local, s, &p);
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
  // tile flags live in the reserved exchange area of every rank (per group)
  o.flag_off = int64_t(group_area(group) + kTileFlagsOff);
  o.cnt_off = int64_t(group_area(group) + kCountersOff);
  o.rows = int(rows);
  o.cols = int(cols);
  o.per = int(cols / W);
  o.tiles_m = p.g.tiles_m;
  o.tiles_n = p.g.tiles_n;
  o.bn = p.bn;
  o.inv_keep = 1.0 - hp->rate;
  o.frate_scale = float(1.0 / (1.0 - hp->rate));
  o.seed = hp->seed;
  o.key = hp->key;
  double th = std::ceil(hp->rate * 9007199254740992.0);
  o.thresh = th <= 0 ? 0 : uint64_t(th);
  o.math = hp->math;
  // every owner adds one arrival per row tile to every rank's counter
  c->mp_arrivals[group] += uint32_t(p.g.tiles_m) * uint32_t(W);
  o.arrive_target = c->mp_arrivals[group];
  for (int i = 0; i < p.g.ranks; ++i)
    p.g.flags[i] = reinterpret_cast<uint32_t*>(p.g.c[i] - o.part_off + o.flag_off);
  p.g.epoch = o.rs.epoch;
  cudaStream_t side;
  cudaEvent_t e0, e1;
  rc = side_stream(c->device, &side, &e0, &e1);
  if (rc) return rc;
  // GEMM on the caller's stream, consumer on a side stream ordered after the
  // caller's prior work; the caller's stream then waits for the consumer.
  CN_CUDA(cudaEventRecord(e0, s));
  CN_CUDA(cudaStreamWaitEvent(side, e0, 0));
  const int nl = local_ranks(c, group);
  int cblocks = std::max(1, std::min(p.g.tiles_m, c->sm_count / nl));
  auto cfn = in_elem == COCONET_BF16 ? overlap_consumer_kernel<__nv_bfloat16> : overlap_consumer_kernel<__half>;
  // The GEMM is enqueued FIRST: it never waits on the consumer, so the pair is
  // deadlock-free whatever the hardware does with the two streams (measured:
  // a consumer enqueued first can hold the GEMM back until it times out). The
  // consumer's CTAs (256 threads, no smem) fit beside the 1-per-SM GEMM CTAs
  // and start polling tile flags while the GEMM is still running.
  rc = launch_tc(c, &p, in_elem, in_elem, c->sm_count, s);
  if (rc) return rc;
  cfn<<<dim3(unsigned(cblocks), unsigned(nl)), 256, 0, side>>>(o);
  CN_CUDA(cudaGetLastError());
  c->launches++;
  CN_CUDA(cudaEventRecord(e1, side));
  CN_CUDA(cudaStreamWaitEvent(s, e1, 0));
  return COCONET_OK;
}

}  // extern "C"
