// Host-side internals of libcoconet_cuda (context, groups, errors, launches).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "coconet_cuda.h"

struct coconet_group_s {
  int first = 0;
  int size = 1;
  uint32_t epoch = 0;  // calls issued on this group (flag value)
};

#include "symm_heap.h"

struct FdServer;

struct coconet_ctx {
  int mode = COCONET_MODE_VIRTUAL;
  int world = 1;
  int rank = 0;  // distributed: this process; virtual: 0
  int device = 0;
  int sm_count = 148;
  size_t heap_bytes = 0;  // per rank, including the reserved pad
  char* heap[coconet::kMaxRanks] = {};
  bool peer_mapped[coconet::kMaxRanks] = {};
  cudaIpcMemHandle_t my_handle{};
  // cuMem heap (heap_kind CUMEM / CUMEM_NVLS, heap_cumem.cu): physical
  // allocation handles (own ranks and imported peers), the exported POSIX
  // descriptor and the socket server that hands it to peers
  int heap_kind = COCONET_HEAP_CUDAMALLOC;
  CUmemGenericAllocationHandle cm_handle[coconet::kMaxRanks] = {};
  bool cm_mapped[coconet::kMaxRanks] = {};
  int cm_fd = -1;
  FdServer* fdsrv = nullptr;
  char peer_srv[coconet::kMaxRanks][64] = {};  // peers' descriptor servers (DISTRIBUTED)
  // NVLS multicast object over the world group's heaps (coconet_nvls_setup)
  CUmemGenericAllocationHandle mc_handle = 0;
  int mc_stage = 0;  // 0 none, 1 created/imported, 2 device added, 3 bound + mapped
  int mc_fd = -1;
  char* mc_base = nullptr;
  SymmHeap alloc;  // user region [kReservedBytes, heap_bytes)
  int* status_host = nullptr;  // host-mapped watchdog word
  int* status_dev = nullptr;
  uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;
  uint64_t launches = 0;
  void* small_dev = nullptr;  // scratch for per-call constants (pointwise)
  size_t small_bytes = 0;
  // cumulative arrivals expected on this rank's per-group counter (overlapped
  // MatMul + fused AllReduce); the device counters start at 0 with the heap
  uint32_t mp_arrivals[coconet::kMaxGroups] = {};
  uint32_t mp_tickets[coconet::kMaxGroups] = {};  // unit tickets handed out so far
  std::vector<coconet_group_s> groups;
  // per-kernel launch facts queried once (the driver queries cost
  // microseconds, more than a small collective's kernel): resident CTAs per
  // SM by (func, threads, smem), and the dynamic smem limit already set
  std::map<std::tuple<const void*, int, size_t>, int> occupancy;
  std::map<const void*, int> smem_set;
};

namespace coconet {

int set_error(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define CN_CUDA(call)                                            \
  do {                                                           \
    cudaError_t _e = (call);                                     \
    if (_e != cudaSuccess) return ::coconet::cuda_fail(_e, #call); \
  } while (0)

// Ranks resident on this device for a launch over `group`.
inline int local_ranks(const coconet_ctx* c, int group) {
  return c->mode == COCONET_MODE_VIRTUAL ? c->groups[size_t(group)].size : 1;
}

// Builds the RankSet for one collective launch on `group` and bumps its epoch.
int make_rankset(coconet_ctx* c, int group, RankSet* rs);

// Heap offset of a caller pointer (own rank's heap; virtual: rank 0's).
int heap_offset(const coconet_ctx* c, const void* p, int64_t* off);

// Blocks per rank for a cooperative launch of `func`.
// Resident CTAs per SM of `func` (cached per context).
int occupancy(coconet_ctx* c, const void* func, int threads, size_t smem, int* per_sm);
// cudaFuncAttributeMaxDynamicSharedMemorySize >= smem (set once per kernel).
int ensure_smem(coconet_ctx* c, const void* func, size_t smem);
int coop_blocks(coconet_ctx* c, const void* func, int threads, size_t smem, int group,
                int64_t want, int* blocks);

int coop_launch(coconet_ctx* c, const void* func, dim3 grid, dim3 block, void** args,
                size_t smem, cudaStream_t stream);

bool valid_group(const coconet_ctx* c, int group);

// cuMem heap (heap_cumem.cu). cumem_create maps a fresh heap for local rank
// slot r; export/import move it between processes as a POSIX descriptor.
int cumem_create(coconet_ctx* c, int r);
int cumem_export(coconet_ctx* c, void* blob_out, size_t* len);
int cumem_import(coconet_ctx* c, const void* blob, size_t len_per_rank);
void cumem_release(coconet_ctx* c);
// heap bytes rounded to what the kind requires (allocation / multicast granularity)
int cumem_round(coconet_ctx* c, size_t* bytes);

}  // namespace coconet
