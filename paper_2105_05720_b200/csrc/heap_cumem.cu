// cuMem-backed symmetric heap and the NVLS multicast object over it.
//
// The default heap is one cudaMalloc per rank shared through CUDA IPC
// (context.cu). This one builds the same heap from the virtual-memory API:
// cuMemCreate (physical pages, exportable as a POSIX descriptor) mapped with
// cuMemAddressReserve / cuMemMap / cuMemSetAccess. Peers import the
// descriptor (fetched over a Unix socket, fdpass.h) and map it into their own
// address space, so heap[q] + off is again rank q's buffer. The reason to
// have it: a multicast object (cuMulticastCreate) can only bind cuMem
// allocations, and with one bound, a kernel reaches ALL ranks' copies of an
// offset through one address: `multimem.ld_reduce` returns the sum over the
// ranks computed in the NVSwitch, `multimem.st` writes every rank (NVLS).
// Reference being replaced: the per-rank vectors of TensorVal
// (state.hpp:17-20) that AllReduce folds (runtime.hpp:384-395).
#include <sys/types.h>
#include <unistd.h>

#include <cstring>
#include <string>

#include "fdpass.h"
#include "internal.h"

using namespace coconet;

namespace {

constexpr uint32_t kBlobMagic = 0x434d454du;  // "CMEM"

// What a rank publishes for its cuMem heap (DISTRIBUTED bootstrap blob).
struct CuMemBlob {
  uint32_t magic;
  int32_t pid;
  uint64_t bytes;
  char server[64];
};

// Driver entry points, resolved through the runtime (cudaGetDriverEntryPoint)
// so the library does not link libcuda directly and still loads where no
// driver is installed (the CPU export checks).
#define CN_DRV_FUNCS(X)                                                                          \
  X(cuGetErrorName) X(cuGetErrorString) X(cuMemAddressReserve) X(cuMemMap) X(cuMemAddressFree)   \
  X(cuMemSetAccess) X(cuMemUnmap) X(cuDeviceGet) X(cuDeviceGetAttribute) X(cuMulticastGetGranularity) \
  X(cuMemGetAllocationGranularity) X(cuMemCreate) X(cuMemRelease) X(cuMemExportToShareableHandle)  \
  X(cuMemImportFromShareableHandle) X(cuMulticastUnbind) X(cuMulticastCreate) X(cuMulticastAddDevice) \
  X(cuMulticastBindMem)

struct DrvApi {
#define CN_X(f) decltype(&::f) f = nullptr;
  CN_DRV_FUNCS(CN_X)
#undef CN_X
  const char* missing = nullptr;  // first entry point the driver did not provide
};

const DrvApi& drv() {
  static const DrvApi d = [] {
    DrvApi t;
#define CN_X(f)                                                                                  \
  {                                                                                              \
    void* p = nullptr;                                                                           \
    cudaDriverEntryPointQueryResult q{};                                                         \
    if (cudaGetDriverEntryPoint(#f, &p, cudaEnableDefault, &q) == cudaSuccess &&                 \
        q == cudaDriverEntryPointSuccess && p)                                                   \
      t.f = reinterpret_cast<decltype(t.f)>(p);                                                  \
    else if (!t.missing)                                                                         \
      t.missing = #f;                                                                            \
  }
    CN_DRV_FUNCS(CN_X)
#undef CN_X
    return t;
  }();
  return d;
}

int drv_check() {
  if (drv().missing)
    return set_error(COCONET_ERR_UNSUPPORTED, std::string("the CUDA driver lacks ") + drv().missing);
  return COCONET_OK;
}

int cu_fail(CUresult r, const char* what) {
  const char* name = nullptr;
  const char* str = nullptr;
  drv().cuGetErrorName(r, &name);
  drv().cuGetErrorString(r, &str);
  return set_error(COCONET_ERR_CUDA, std::string(what) + ": " + (name ? name : "?") + " (" + (str ? str : "") + ")");
}

#define CN_CU(call)                                  \
  do {                                               \
    CUresult _r = (call);                            \
    if (_r != CUDA_SUCCESS) return cu_fail(_r, #call); \
  } while (0)

CUmemAllocationProp heap_prop(int device) {
  CUmemAllocationProp p{};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return p;
}

// Reserves and maps `h` (bytes) read/write for `device`.
int map_handle(CUmemGenericAllocationHandle h, size_t bytes, int device, char** out) {
  CUdeviceptr va = 0;
  CN_CU(drv().cuMemAddressReserve(&va, bytes, 0, 0, 0));
  CUresult r = drv().cuMemMap(va, bytes, 0, h, 0);
  if (r != CUDA_SUCCESS) {
    drv().cuMemAddressFree(va, bytes);
    return cu_fail(r, "cuMemMap");
  }
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = drv().cuMemSetAccess(va, bytes, &acc, 1);
  if (r != CUDA_SUCCESS) {
    drv().cuMemUnmap(va, bytes);
    drv().cuMemAddressFree(va, bytes);
    return cu_fail(r, "cuMemSetAccess");
  }
  *out = reinterpret_cast<char*>(va);
  return COCONET_OK;
}

// Why multicast cannot be used on `device`, or nullptr.
const char* nvls_blocker(int device, int world) {
  if (drv().missing) return "the CUDA driver lacks the multicast entry points";
  CUdevice d;
  if (drv().cuDeviceGet(&d, device) != CUDA_SUCCESS) return "cuDeviceGet failed";
  int mc = 0;
  if (drv().cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d) != CUDA_SUCCESS || !mc)
    return "CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED is 0 (no NVSwitch multicast: single GPU, no fabric manager, or "
           "the nvswitch devices are not mapped into this container)";
  CUmulticastObjectProp p{};
  p.numDevices = unsigned(world);
  p.size = size_t(2) << 20;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g = 0;
  if (drv().cuMulticastGetGranularity(&g, &p, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS || g == 0)
    return "cuMulticastGetGranularity failed";
  // the attribute can be 1 where the fabric is absent (a one-GPU slice of an
  // NVSwitch node): only a created object proves multicast works
  p.size = g;
  CUmemGenericAllocationHandle h = 0;
  if (drv().cuMulticastCreate(&h, &p) != CUDA_SUCCESS)
    return "cuMulticastCreate fails (the NVSwitch fabric is not reachable from this process: e.g. only "
           "/dev/nvidia0 is mapped, no nvidia-nvswitch / IMEX devices)";
  drv().cuMemRelease(h);
  return nullptr;
}

}  // namespace

namespace coconet {

int cumem_round(coconet_ctx* c, size_t* bytes) {
  cudaFree(nullptr);  // the runtime's primary context is current for the driver calls
  if (int rc = drv_check()) return rc;
  const CUmemAllocationProp p = heap_prop(c->device);
  size_t g = 0;
  CN_CU(drv().cuMemGetAllocationGranularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  if (c->heap_kind == COCONET_HEAP_CUMEM_NVLS) {
    if (const char* why = nvls_blocker(c->device, c->world))
      return set_error(COCONET_ERR_UNSUPPORTED, std::string("NVLS heap: ") + why);
    CUmulticastObjectProp mp{};
    mp.numDevices = unsigned(c->world);
    mp.size = *bytes;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t mg = 0;
    CN_CU(drv().cuMulticastGetGranularity(&mg, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    if (mg > g) g = (mg / g) * g == mg ? mg : mg * g;
  }
  *bytes = (*bytes + g - 1) / g * g;
  return COCONET_OK;
}

int cumem_create(coconet_ctx* c, int r) {
  const CUmemAllocationProp p = heap_prop(c->device);
  CUmemGenericAllocationHandle h = 0;
  CN_CU(drv().cuMemCreate(&h, c->heap_bytes, &p, 0));
  char* va = nullptr;
  int rc = map_handle(h, c->heap_bytes, c->device, &va);
  if (rc) {
    drv().cuMemRelease(h);
    return rc;
  }
  c->cm_handle[r] = h;
  c->cm_mapped[r] = true;
  c->heap[r] = va;
  return COCONET_OK;
}

int cumem_export(coconet_ctx* c, void* blob_out, size_t* len) {
  if (len) {
    if (blob_out && *len < sizeof(CuMemBlob)) return set_error(COCONET_ERR_INVALID_INPUT, "handle buffer too small");
    *len = sizeof(CuMemBlob);
  }
  if (!blob_out) return COCONET_OK;
  if (c->cm_fd < 0) {
    int fd = -1;
    CN_CU(drv().cuMemExportToShareableHandle(&fd, c->cm_handle[c->rank], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    c->cm_fd = fd;
  }
  if (!c->fdsrv) {
    c->fdsrv = new FdServer();
    if (!c->fdsrv->start("coconet")) {
      delete c->fdsrv;
      c->fdsrv = nullptr;
      return set_error(COCONET_ERR_CUDA, "cannot start the heap descriptor server (abstract Unix socket)");
    }
  }
  c->fdsrv->set(0, c->cm_fd);
  CuMemBlob b{};
  b.magic = kBlobMagic;
  b.pid = int32_t(getpid());
  b.bytes = c->heap_bytes;
  std::strncpy(b.server, c->fdsrv->name, sizeof(b.server) - 1);
  std::memcpy(blob_out, &b, sizeof(b));
  return COCONET_OK;
}

int cumem_import(coconet_ctx* c, const void* all, size_t len_per_rank) {
  if (len_per_rank != sizeof(CuMemBlob)) return set_error(COCONET_ERR_INVALID_INPUT, "bad handle length (cuMem heap)");
  const char* blob = static_cast<const char*>(all);
  for (int r = 0; r < c->world; ++r) {
    CuMemBlob b;
    std::memcpy(&b, blob + size_t(r) * len_per_rank, sizeof(b));
    if (b.magic != kBlobMagic)
      return set_error(COCONET_ERR_INVALID_INPUT, "rank " + std::to_string(r) + " did not publish a cuMem heap");
    if (b.bytes != c->heap_bytes)
      return set_error(COCONET_ERR_INVALID_INPUT, "heap sizes differ across ranks");
    std::memcpy(c->peer_srv[r], b.server, sizeof(b.server));
    if (r == c->rank || c->heap[r]) continue;
    const char* why = "";
    const int fd = fd_fetch(b.server, 0, 30000, &why);
    if (fd < 0) return set_error(COCONET_ERR_CUDA, std::string("heap descriptor of rank ") + std::to_string(r) + ": " + why);
    CUmemGenericAllocationHandle h = 0;
    CUresult res = drv().cuMemImportFromShareableHandle(&h, reinterpret_cast<void*>(uintptr_t(fd)),
                                                  CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close(fd);
    if (res != CUDA_SUCCESS) return cu_fail(res, "cuMemImportFromShareableHandle");
    char* va = nullptr;
    int rc = map_handle(h, c->heap_bytes, c->device, &va);
    if (rc) {
      drv().cuMemRelease(h);
      return rc;
    }
    c->cm_handle[r] = h;
    c->cm_mapped[r] = true;
    c->heap[r] = va;
  }
  return COCONET_OK;
}

void cumem_release(coconet_ctx* c) {
  if (c->heap_kind == COCONET_HEAP_CUDAMALLOC) return;
  if (c->fdsrv) {
    c->fdsrv->stop();
    delete c->fdsrv;
    c->fdsrv = nullptr;
  }
  if (c->mc_base) {
    drv().cuMemUnmap(reinterpret_cast<CUdeviceptr>(c->mc_base), c->heap_bytes);
    drv().cuMemAddressFree(reinterpret_cast<CUdeviceptr>(c->mc_base), c->heap_bytes);
    c->mc_base = nullptr;
  }
  if (c->mc_stage >= 3) {
    CUdevice d;
    if (drv().cuDeviceGet(&d, c->device) == CUDA_SUCCESS) drv().cuMulticastUnbind(c->mc_handle, d, 0, c->heap_bytes);
  }
  if (c->mc_stage >= 1) drv().cuMemRelease(c->mc_handle);
  c->mc_stage = 0;
  if (c->mc_fd >= 0) close(c->mc_fd);
  c->mc_fd = -1;
  for (int r = 0; r < kMaxRanks; ++r) {
    if (!c->cm_mapped[r]) continue;
    const CUdeviceptr va = reinterpret_cast<CUdeviceptr>(c->heap[r]);
    drv().cuMemUnmap(va, c->heap_bytes);
    drv().cuMemAddressFree(va, c->heap_bytes);
    drv().cuMemRelease(c->cm_handle[r]);
    c->cm_mapped[r] = false;
    c->heap[r] = nullptr;
  }
  if (c->cm_fd >= 0) close(c->cm_fd);
  c->cm_fd = -1;
}

}  // namespace coconet

extern "C" {

int coconet_heap_kind(coconet_ctx_t c) { return c ? c->heap_kind : -1; }

int coconet_nvls_supported(int device, int world, char* why, size_t why_len) {
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaFree(nullptr);
  const char* b = e != cudaSuccess ? "no CUDA device" : nvls_blocker(device, world < 1 ? 1 : world);
  if (why && why_len) {
    std::strncpy(why, b ? b : "", why_len - 1);
    why[why_len - 1] = '\0';
  }
  return b ? 0 : 1;
}

// Collective NVLS bootstrap, DISTRIBUTED world group, heap kind CUMEM_NVLS,
// after coconet_open_peers; the caller puts a process barrier between the
// stages (cuMulticastAddDevice must have run on every rank before any rank
// binds memory):
//   stage 0: rank 0 creates the multicast object and serves its descriptor
//   stage 1: the other ranks import it; every rank adds its device
//   stage 2: every rank binds its heap and maps the multicast address range
int coconet_nvls_setup(coconet_ctx_t c, int stage) {
  if (!c) return set_error(COCONET_ERR_INVALID_INPUT, "null ctx");
  if (c->heap_kind != COCONET_HEAP_CUMEM_NVLS || c->mode != COCONET_MODE_DISTRIBUTED)
    return set_error(COCONET_ERR_UNSUPPORTED, "NVLS needs a DISTRIBUTED context with heap kind COCONET_HEAP_CUMEM_NVLS");
  if (stage != c->mc_stage) return set_error(COCONET_ERR_INVALID_INPUT, "NVLS setup stages run 0, 1, 2 in order");
  CUdevice dev;
  CN_CU(drv().cuDeviceGet(&dev, c->device));
  if (stage == 0) {
    if (c->rank == 0) {
      if (!c->fdsrv) return set_error(COCONET_ERR_INVALID_INPUT, "call coconet_open_peers before coconet_nvls_setup");
      CUmulticastObjectProp p{};
      p.numDevices = unsigned(c->world);
      p.size = c->heap_bytes;
      p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
      CN_CU(drv().cuMulticastCreate(&c->mc_handle, &p));
      int fd = -1;
      CUresult r = drv().cuMemExportToShareableHandle(&fd, c->mc_handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
      if (r != CUDA_SUCCESS) {
        drv().cuMemRelease(c->mc_handle);
        return cu_fail(r, "cuMemExportToShareableHandle(multicast)");
      }
      c->mc_fd = fd;
      c->fdsrv->set(1, fd);
      c->mc_stage = 1;
    } else {
      c->mc_stage = 1;  // imported in stage 1, once rank 0 serves it
    }
    return COCONET_OK;
  }
  if (stage == 1) {
    if (c->rank != 0) {
      const char* why = "";
      const int fd = fd_fetch(c->peer_srv[0], 1, 30000, &why);
      if (fd < 0) return set_error(COCONET_ERR_CUDA, std::string("multicast descriptor of rank 0: ") + why);
      CUresult r = drv().cuMemImportFromShareableHandle(&c->mc_handle, reinterpret_cast<void*>(uintptr_t(fd)),
                                                  CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
      close(fd);
      if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemImportFromShareableHandle(multicast)");
    }
    CN_CU(drv().cuMulticastAddDevice(c->mc_handle, dev));
    c->mc_stage = 2;
    return COCONET_OK;
  }
  CN_CU(drv().cuMulticastBindMem(c->mc_handle, 0, c->cm_handle[c->rank], 0, c->heap_bytes, 0));
  c->mc_stage = 3;
  char* va = nullptr;
  int rc = map_handle(c->mc_handle, c->heap_bytes, c->device, &va);
  if (rc) return rc;
  c->mc_base = va;
  return COCONET_OK;
}

int coconet_nvls_mapped(coconet_ctx_t c) { return c && c->mc_base ? 1 : 0; }

}  // extern "C"
