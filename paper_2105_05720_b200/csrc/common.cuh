// Device-side building blocks shared by every kernel of libcoconet_cuda.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "coconet_cuda.h"

namespace coconet {

constexpr int kMaxRanks = COCONET_MAX_RANKS;
constexpr int kMaxBlocks = 2048;   // per rank per launch (flag slots)
constexpr int kMaxGroups = 4;
constexpr int kFlagPhases = 8;     // distinct barrier slots per launch
// signal pad at the start of every rank's heap:
//   uint32 flags[kMaxGroups][kFlagPhases][kMaxRanks][kMaxBlocks]
constexpr size_t kPadBytes =
    size_t(kMaxGroups) * kFlagPhases * kMaxRanks * kMaxBlocks * sizeof(uint32_t);
// per-group areas after the pad (kGroupAreaBytes each):
//   [0, kTileFlagsOff)              LAMB per-tensor partials exchange
//   [kTileFlagsOff, kCountersOff)   per-tile flags of the overlapped MatMul
//   [kCountersOff, kGroupAreaBytes) arrival counters
constexpr size_t kXchBytes = size_t(8) << 20;
constexpr size_t kGroupAreaBytes = kXchBytes / kMaxGroups;
constexpr size_t kTileFlagsOff = kGroupAreaBytes - (size_t(128) << 10);
constexpr size_t kCountersOff = kGroupAreaBytes - (size_t(64) << 10);
constexpr size_t kReservedBytes = kPadBytes + kXchBytes;

__host__ __device__ constexpr size_t group_area(int group) {
  return kPadBytes + size_t(group) * kGroupAreaBytes;
}

// Per-launch view of the ranks a kernel touches. Virtual mode: all ranks of
// the group are on this device, blockIdx.y = group rank. Distributed: one
// rank, blockIdx.y = 0 and `me` is the group rank.
struct RankSet {
  char* base[kMaxRanks];  // heap base of every group rank (peer-mapped when distributed)
  int world;              // group size W
  int me;                 // distributed: own group rank; virtual: -1
  int group;              // group id (flag region)
  uint32_t epoch;         // per-group call counter (flag value of this launch)
  char* mc;               // NVLS multicast view of every rank's heap (world group), or null
  int* status;            // host-mapped status word (watchdog)
  unsigned long long timeout_ns;

  __device__ __forceinline__ int rank() const { return me >= 0 ? me : int(blockIdx.y); }
};

// ---------------------------------------------------------------------------
// Counter PRNG, bit-exact with ccopt::counter_uniform (expr.hpp:15-23).

__host__ __device__ __forceinline__ uint64_t prng_bits(uint64_t seed, uint64_t key,
                                                       uint64_t index) {
  uint64_t x = seed ^ (key * 0x9e3779b97f4a7c15ull) ^ (index + 0x632be59bd9b4e019ull);
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x >> 11;  // the 53-bit mantissa numerator
}

__host__ __device__ __forceinline__ double counter_uniform(uint64_t seed, uint64_t key,
                                                           uint64_t index) {
  return double(prng_bits(seed, key, index)) * (1.0 / 9007199254740992.0);
}

// dropout_keep (expr.hpp:25-27): u >= rate  <=>  bits >= ceil(rate * 2^53),
// exact because the scaling is a power of two. `thresh` is precomputed on the
// host as the smallest integer k with k * 2^-53 >= rate.
__device__ __forceinline__ bool dropout_keep_bits(uint64_t seed, uint64_t key, uint64_t index,
                                                  uint64_t thresh) {
  return prng_bits(seed, key, index) >= thresh;
}

// ---------------------------------------------------------------------------
// Element conversions.

template <int E> struct ElemT;
template <> struct ElemT<COCONET_F32> { using T = float; };
template <> struct ElemT<COCONET_F16> { using T = __half; };
template <> struct ElemT<COCONET_BF16> { using T = __nv_bfloat16; };

__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__half x) { return __half2float(x); }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f32(float x);
template <> __device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ __half from_f32<__half>(float x) { return __float2half_rn(x); }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// 4-element vectors: fp32 -> 16 B, 16-bit -> 8 B.
template <typename T> struct Vec4 { T v[4]; };

template <typename T>
__device__ __forceinline__ void load4(const T* p, float out[4]) {
  if constexpr (sizeof(T) == 4) {
    float4 x = __ldg(reinterpret_cast<const float4*>(p));
    out[0] = x.x; out[1] = x.y; out[2] = x.z; out[3] = x.w;
  } else {
    uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
    const T* h = reinterpret_cast<const T*>(&x);
    out[0] = to_f32(h[0]); out[1] = to_f32(h[1]); out[2] = to_f32(h[2]); out[3] = to_f32(h[3]);
  }
}

// Plain (coherent) loads for data that other ranks write during the kernel.
template <typename T>
__device__ __forceinline__ void load4_cg(const T* p, float out[4]) {
  if constexpr (sizeof(T) == 4) {
    float4 x = __ldcg(reinterpret_cast<const float4*>(p));
    out[0] = x.x; out[1] = x.y; out[2] = x.z; out[3] = x.w;
  } else {
    uint2 x = __ldcg(reinterpret_cast<const uint2*>(p));
    const T* h = reinterpret_cast<const T*>(&x);
    out[0] = to_f32(h[0]); out[1] = to_f32(h[1]); out[2] = to_f32(h[2]); out[3] = to_f32(h[3]);
  }
}

template <typename T>
__device__ __forceinline__ void store4(T* p, const float in[4]) {
  if constexpr (sizeof(T) == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(in[0], in[1], in[2], in[3]);
  } else {
    T h[4] = {from_f32<T>(in[0]), from_f32<T>(in[1]), from_f32<T>(in[2]), from_f32<T>(in[3])};
    *reinterpret_cast<uint2*>(p) = *reinterpret_cast<const uint2*>(h);
  }
}

// ---------------------------------------------------------------------------
// Cross-rank flags: release/acquire at system scope so NVLink peers (and, in
// virtual mode, co-resident CTAs standing in for them) observe the data written
// before the flag.

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t* flag_slot(char* heap, int group, int phase, int src,
                                               int block) {
  uint32_t* pad = reinterpret_cast<uint32_t*>(heap);
  return pad + ((size_t(group) * kFlagPhases + phase) * kMaxRanks + src) * kMaxBlocks + block;
}

// Spin until *p >= want (wrap-safe). Returns false on watchdog expiry after
// recording COCONET_ERR_TIMEOUT in the host-mapped status word.
__device__ __forceinline__ bool wait_flag(const uint32_t* p, uint32_t want, const RankSet& rs) {
  if (int32_t(ld_acquire_sys(p) - want) >= 0) return true;
  unsigned long long t0 = globaltimer();
  int spins = 0;
  while (int32_t(ld_acquire_sys(p) - want) < 0) {
    if (++spins > 64) __nanosleep(64);
    if ((spins & 255) == 0 && globaltimer() - t0 > rs.timeout_ns) {
      atomicCAS(rs.status, 0, COCONET_ERR_TIMEOUT);
      return false;
    }
  }
  return true;
}

// Pairwise barrier between this CTA and the CTA with the same blockIdx.x on
// every other rank of the group: thread q < W signals rank q and waits for
// rank q. `fence` orders this CTA's prior (remote) writes before the signal.
// The waiter resets the slot it consumed to 0, so a slot is always 0 before
// its next use (the peer's next signal into it comes only after this rank
// reached a later barrier of the same launch, or the entry barrier of the
// next one; every barrier of a launch uses its own phase). The protocol
// therefore does not depend on the host's epoch advancing: a launch
// captured in a CUDA graph replays correctly with its baked-in epoch.
__device__ __forceinline__ bool rank_barrier(const RankSet& rs, int phase) {
  if (rs.world == 1) {  // no peer to meet
    __syncthreads();
    return true;
  }
  __syncthreads();
  bool ok = true;
  const int me = rs.rank();
  const int q = threadIdx.x;
  if (q < rs.world) {
    __threadfence_system();
    st_release_sys(flag_slot(rs.base[q], rs.group, phase, me, blockIdx.x), rs.epoch);
    uint32_t* mine = flag_slot(rs.base[me], rs.group, phase, q, blockIdx.x);
    ok = wait_flag(mine, rs.epoch, rs);
    if (ok) *reinterpret_cast<volatile uint32_t*>(mine) = 0u;  // consumed
  }
  return __syncthreads_and(ok);
}

// Entry / exit barrier of a kernel whose ranks touch disjoint data inside the
// launch (each rank reads every peer's input chunk r and writes chunk r of
// every peer's output). It orders the launch against the peers' producers
// before and consumers after it, which only separate processes need: in
// VIRTUAL mode every rank is a slice of this grid and stream order already
// does it, so the CTA only syncs its own threads.
__device__ __forceinline__ bool edge_barrier(const RankSet& rs, int phase) {
  if (rs.me < 0) {
    __syncthreads();
    return true;
  }
  return rank_barrier(rs, phase);
}

__device__ __forceinline__ bool failed(const RankSet& rs) {
  return *reinterpret_cast<volatile int*>(rs.status) != 0;
}

}  // namespace coconet
