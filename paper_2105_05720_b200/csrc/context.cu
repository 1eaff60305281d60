// Context, symmetric heap, process groups and error plumbing of
// libcoconet_cuda.
//
// Replaces the reference's in-process rank model: ccopt keeps one host
// vector per rank (TensorVal::per_rank, state.hpp:17-20) and "sends" by
// copying between them (runtime.hpp:306-350). Here every rank owns a device
// heap of identical size; symmetric buffers share one offset on all ranks, so
// a kernel reaches rank q's copy as heap[q] + offset — a local address in
// VIRTUAL mode, an NVLink peer mapping (CUDA IPC) in DISTRIBUTED mode.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "internal.h"

using namespace coconet;

namespace {
thread_local std::string g_last_error;
}

namespace coconet {

int set_error(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char* what) {
  return set_error(COCONET_ERR_CUDA,
                   std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

bool valid_group(const coconet_ctx* c, int group) {
  return c && group >= 0 && size_t(group) < c->groups.size();
}

int make_rankset(coconet_ctx* c, int group, RankSet* rs) {
  if (!valid_group(c, group)) return set_error(COCONET_ERR_NO_SUCH_RANK, "no such group");
  coconet_group_s& g = c->groups[size_t(group)];
  std::memset(rs, 0, sizeof(*rs));
  for (int i = 0; i < g.size; ++i) {
    int wr = g.first + i;
    if (!c->heap[wr]) return set_error(COCONET_ERR_NO_SUCH_RANK, "peer heap of rank " + std::to_string(wr) + " is not mapped");
    rs->base[i] = c->heap[wr];
  }
  rs->world = g.size;
  if (c->mode == COCONET_MODE_VIRTUAL) {
    rs->me = -1;
  } else {
    if (c->rank < g.first || c->rank >= g.first + g.size)
      return set_error(COCONET_ERR_NO_SUCH_RANK, "this rank is not a member of the group");
    rs->me = c->rank - g.first;
  }
  rs->group = group;
  rs->epoch = ++g.epoch;
  if (rs->epoch == 0) rs->epoch = ++g.epoch;  // 0 is the "never signalled" value
  // the multicast range spans the world group's heaps only
  rs->mc = group == 0 && c->mc_base ? c->mc_base : nullptr;
  rs->status = c->status_dev;
  rs->timeout_ns = c->timeout_ns;
  return COCONET_OK;
}

int heap_offset(const coconet_ctx* c, const void* p, int64_t* off) {
  const char* base = c->heap[c->mode == COCONET_MODE_VIRTUAL ? 0 : c->rank];
  const char* q = static_cast<const char*>(p);
  if (!p || q < base + kReservedBytes || q >= base + c->heap_bytes)
    return set_error(COCONET_ERR_INVALID_INPUT,
                     "pointer is not inside this rank's symmetric heap (use coconet_symm_alloc)");
  *off = q - base;
  return COCONET_OK;
}

int occupancy(coconet_ctx* c, const void* func, int threads, size_t smem, int* per_sm) {
  const auto key = std::make_tuple(func, threads, smem);
  auto it = c->occupancy.find(key);
  if (it == c->occupancy.end()) {
    int n = 0;
    CN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, func, threads, smem));
    it = c->occupancy.emplace(key, n).first;
  }
  *per_sm = it->second;
  return COCONET_OK;
}

int ensure_smem(coconet_ctx* c, const void* func, size_t smem) {
  auto it = c->smem_set.find(func);
  if (it != c->smem_set.end() && size_t(it->second) >= smem) return COCONET_OK;
  CN_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  c->smem_set[func] = int(smem);
  return COCONET_OK;
}

int coop_blocks(coconet_ctx* c, const void* func, int threads, size_t smem, int group,
                int64_t want, int* blocks) {
  int per_sm = 0;
  int rc = occupancy(c, func, threads, smem, &per_sm);
  if (rc) return rc;
  if (per_sm < 1) return set_error(COCONET_ERR_CUDA, "kernel cannot be resident (occupancy 0)");
  int64_t cap = int64_t(per_sm) * c->sm_count / local_ranks(c, group);
  if (cap > kMaxBlocks) cap = kMaxBlocks;
  int64_t b = want < cap ? want : cap;
  if (b < 1) b = 1;
  *blocks = int(b);
  return COCONET_OK;
}

int coop_launch(coconet_ctx* c, const void* func, dim3 grid, dim3 block, void** args,
                size_t smem, cudaStream_t stream) {
  CN_CUDA(cudaLaunchCooperativeKernel(func, grid, block, args, smem, stream));
  c->launches++;
  return COCONET_OK;
}

}  // namespace coconet

extern "C" {

const char* coconet_last_error(void) { return g_last_error.c_str(); }

const char* coconet_status_name(int s) {
  switch (s) {
    case COCONET_OK: return "OK";
    case COCONET_ERR_LAYOUT_MISMATCH: return "LayoutMismatch";
    case COCONET_ERR_SHAPE_MISMATCH: return "ShapeMismatch";
    case COCONET_ERR_INVALID_INPUT: return "InvalidInput";
    case COCONET_ERR_NO_SUCH_RANK: return "NoSuchRank";
    case COCONET_ERR_OPERAND_LAYOUT_MISMATCH: return "OperandLayoutMismatch";
    case COCONET_ERR_DIVISIBILITY: return "DivisibilityError";
    case COCONET_ERR_REPLICATION_VIOLATION: return "ReplicationViolation";
    case COCONET_ERR_UNKNOWN_ID: return "UnknownId";
    case COCONET_ERR_CUDA: return "CudaError";
    case COCONET_ERR_TIMEOUT: return "Timeout";
    case COCONET_ERR_UNSUPPORTED: return "Unsupported";
    case COCONET_ERR_OOM: return "OutOfHeap";
    default: return "Unknown";
  }
}

int coconet_init(coconet_ctx_t* out, int mode, int rank, int world, int device,
                 size_t heap_bytes_per_rank) {
  return coconet_init_ex(out, mode, rank, world, device, heap_bytes_per_rank, COCONET_HEAP_DEFAULT);
}

int coconet_init_ex(coconet_ctx_t* out, int mode, int rank, int world, int device,
                    size_t heap_bytes_per_rank, int heap_kind) {
  if (!out) return set_error(COCONET_ERR_INVALID_INPUT, "null ctx out");
  if (heap_kind == COCONET_HEAP_DEFAULT) {  // COCONET_HEAP=cumem|nvls|cudamalloc
    const char* e = getenv("COCONET_HEAP");
    heap_kind = !e ? COCONET_HEAP_CUDAMALLOC
                : !strcmp(e, "cumem") ? COCONET_HEAP_CUMEM
                : !strcmp(e, "nvls") ? COCONET_HEAP_CUMEM_NVLS
                                     : COCONET_HEAP_CUDAMALLOC;
  }
  if (heap_kind < COCONET_HEAP_CUDAMALLOC || heap_kind > COCONET_HEAP_CUMEM_NVLS)
    return set_error(COCONET_ERR_INVALID_INPUT, "unknown heap kind");
  if (heap_kind == COCONET_HEAP_CUMEM_NVLS && mode != COCONET_MODE_DISTRIBUTED)
    return set_error(COCONET_ERR_UNSUPPORTED, "an NVLS heap spans one GPU per rank (DISTRIBUTED mode)");
  *out = nullptr;
  if (world < 1 || world > kMaxRanks)
    return set_error(COCONET_ERR_NO_SUCH_RANK, "world size must be in [1, " + std::to_string(kMaxRanks) + "]");
  if (mode != COCONET_MODE_VIRTUAL && mode != COCONET_MODE_DISTRIBUTED)
    return set_error(COCONET_ERR_INVALID_INPUT, "unknown mode");
  if (mode == COCONET_MODE_DISTRIBUTED && (rank < 0 || rank >= world))
    return set_error(COCONET_ERR_NO_SUCH_RANK, "rank out of range");
  auto* c = new coconet_ctx();
  c->mode = mode;
  c->world = world;
  c->rank = mode == COCONET_MODE_VIRTUAL ? 0 : rank;
  c->device = device;
  c->heap_kind = heap_kind;
  c->heap_bytes = ((heap_bytes_per_rank + kReservedBytes + 4095) / 4096) * 4096;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaSetDevice");
  }
  const bool cumem = heap_kind != COCONET_HEAP_CUDAMALLOC;
  if (cumem) {
    int rc = cumem_round(c, &c->heap_bytes);
    if (rc) {
      delete c;
      return rc;
    }
  }
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  int nlocal = mode == COCONET_MODE_VIRTUAL ? world : 1;
  for (int i = 0; i < nlocal; ++i) {
    int r = mode == COCONET_MODE_VIRTUAL ? i : rank;
    if (cumem) {
      int rc = cumem_create(c, r);
      if (rc) {
        coconet_finalize(c);
        return rc;
      }
      e = cudaMemset(c->heap[r], 0, kReservedBytes);
    } else {
      e = cudaMalloc(&c->heap[r], c->heap_bytes);
      if (e == cudaSuccess) e = cudaMemset(c->heap[r], 0, kReservedBytes);
    }
    if (e != cudaSuccess) {
      coconet_finalize(c);
      return cuda_fail(e, "heap cudaMalloc");
    }
  }
  e = cudaHostAlloc(&c->status_host, sizeof(int), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(&c->status_dev, c->status_host, 0);
  if (e != cudaSuccess) {
    coconet_finalize(c);
    return cuda_fail(e, "status cudaHostAlloc");
  }
  *c->status_host = 0;
  if (mode == COCONET_MODE_DISTRIBUTED && !cumem) {
    e = cudaIpcGetMemHandle(&c->my_handle, c->heap[rank]);
    if (e != cudaSuccess) {
      coconet_finalize(c);
      return cuda_fail(e, "cudaIpcGetMemHandle");
    }
  }
  coconet_group_s world_group;
  world_group.first = 0;
  world_group.size = world;
  c->groups.push_back(world_group);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    coconet_finalize(c);
    return cuda_fail(e, "init sync");
  }
  *out = c;
  return COCONET_OK;
}

int coconet_finalize(coconet_ctx_t c) {
  if (!c) return COCONET_OK;
  cudaDeviceSynchronize();
  cumem_release(c);  // cuMem heaps and the multicast mapping (no-op otherwise)
  for (int r = 0; r < kMaxRanks; ++r) {
    if (!c->heap[r]) continue;
    if (c->peer_mapped[r])
      cudaIpcCloseMemHandle(c->heap[r]);
    else
      cudaFree(c->heap[r]);
  }
  if (c->status_host) cudaFreeHost(c->status_host);
  if (c->small_dev) cudaFree(c->small_dev);
  delete c;
  return COCONET_OK;
}

int coconet_world(coconet_ctx_t c, int* world, int* rank, int* mode) {
  if (!c) return set_error(COCONET_ERR_INVALID_INPUT, "null ctx");
  if (world) *world = c->world;
  if (rank) *rank = c->rank;
  if (mode) *mode = c->mode;
  return COCONET_OK;
}

int coconet_heap_handle(coconet_ctx_t c, void* handle_out, size_t* len) {
  if (!c || c->mode != COCONET_MODE_DISTRIBUTED)
    return set_error(COCONET_ERR_INVALID_INPUT, "heap handles exist in DISTRIBUTED mode only");
  if (c->heap_kind != COCONET_HEAP_CUDAMALLOC) return cumem_export(c, handle_out, len);
  if (len) {
    if (handle_out && *len < sizeof(cudaIpcMemHandle_t))
      return set_error(COCONET_ERR_INVALID_INPUT, "handle buffer too small");
    *len = sizeof(cudaIpcMemHandle_t);
  }
  if (handle_out) std::memcpy(handle_out, &c->my_handle, sizeof(cudaIpcMemHandle_t));
  return COCONET_OK;
}

int coconet_open_peers(coconet_ctx_t c, const void* all, size_t len_per_rank) {
  if (!c || c->mode != COCONET_MODE_DISTRIBUTED)
    return set_error(COCONET_ERR_INVALID_INPUT, "open_peers is DISTRIBUTED-only");
  if (c->heap_kind != COCONET_HEAP_CUDAMALLOC) return cumem_import(c, all, len_per_rank);
  if (len_per_rank != sizeof(cudaIpcMemHandle_t))
    return set_error(COCONET_ERR_INVALID_INPUT, "bad handle length");
  const char* blob = static_cast<const char*>(all);
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank || c->heap[r]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, blob + size_t(r) * len_per_rank, sizeof(h));
    void* p = nullptr;
    CN_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->heap[r] = static_cast<char*>(p);
    c->peer_mapped[r] = true;
  }
  return COCONET_OK;
}

int coconet_symm_alloc(coconet_ctx_t c, size_t bytes, size_t* offset) {
  if (!c || !offset) return set_error(COCONET_ERR_INVALID_INPUT, "null argument");
  if (c->alloc.end == 0) c->alloc.init(kReservedBytes, c->heap_bytes);
  if (!c->alloc.alloc(bytes, offset))
    return set_error(COCONET_ERR_OOM, "symmetric heap exhausted: need " + std::to_string((bytes + 255) & ~size_t(255)) +
                                          " bytes, largest free block " + std::to_string(c->alloc.largest_free()) +
                                          " of " + std::to_string(c->heap_bytes));
  return COCONET_OK;
}

int coconet_symm_free(coconet_ctx_t c, size_t offset) {
  if (!c) return set_error(COCONET_ERR_INVALID_INPUT, "null ctx");
  if (!c->alloc.release(offset))
    return set_error(COCONET_ERR_INVALID_INPUT, "offset " + std::to_string(offset) + " is not a live symmetric allocation");
  return COCONET_OK;
}

int coconet_symm_reset(coconet_ctx_t c) {
  if (!c) return set_error(COCONET_ERR_INVALID_INPUT, "null ctx");
  c->alloc.init(kReservedBytes, c->heap_bytes);
  return COCONET_OK;
}

size_t coconet_symm_high_water(coconet_ctx_t c) { return c ? c->alloc.high : 0; }

size_t coconet_heap_bytes(coconet_ctx_t c) { return c ? c->heap_bytes : 0; }

void* coconet_symm_ptr(coconet_ctx_t c, int rank, size_t offset) {
  if (!c || rank < 0 || rank >= c->world || !c->heap[rank] || offset >= c->heap_bytes) return nullptr;
  return c->heap[rank] + offset;
}

int coconet_group_create(coconet_ctx_t c, int first_rank, int size, int* group) {
  if (!c) return set_error(COCONET_ERR_INVALID_INPUT, "null ctx");
  if (first_rank < 0 || size < 1 || first_rank + size > c->world)
    return set_error(COCONET_ERR_NO_SUCH_RANK, "group outside the world");
  if (int(c->groups.size()) >= kMaxGroups)
    return set_error(COCONET_ERR_UNSUPPORTED, "too many groups");
  coconet_group_s g;
  g.first = first_rank;
  g.size = size;
  c->groups.push_back(g);
  if (group) *group = int(c->groups.size()) - 1;
  return COCONET_OK;
}

int coconet_check(coconet_ctx_t c, void* stream) {
  if (!c) return set_error(COCONET_ERR_INVALID_INPUT, "null ctx");
  CN_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  int s = *reinterpret_cast<volatile int*>(c->status_host);
  if (s != 0) {
    *c->status_host = 0;
    return set_error(s, std::string("device reported ") + coconet_status_name(s) +
                            " (a peer rank never arrived at a flag barrier)");
  }
  return COCONET_OK;
}

int coconet_set_timeout_ms(coconet_ctx_t c, uint32_t ms) {
  if (!c) return set_error(COCONET_ERR_INVALID_INPUT, "null ctx");
  c->timeout_ns = uint64_t(ms) * 1000000ull;
  return COCONET_OK;
}

uint64_t coconet_launch_count(coconet_ctx_t c) { return c ? c->launches : 0; }

}  // extern "C"
