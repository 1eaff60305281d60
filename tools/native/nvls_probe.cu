// Capability probe (not product code): does this box's driver / fabric
// support multicast objects (NVLS) and POSIX-FD cuMem handles? Creates a
// one-device multicast object, binds a cuMem allocation, maps it, and runs
// multimem.ld_reduce / multimem.st through it.
#include <cuda.h>
#include <cstdio>
#include <cstring>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); \
  printf("FAIL %s: %s\n", #x, s_); return 1; } } while (0)

__global__ void mm_kernel(float* mc, float* uc, float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i * 4 >= n) return;
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(mc + 4 * i) : "memory");
  reinterpret_cast<float4*>(out)[i] = v;
  float4 w = make_float4(v.x * 2, v.y * 2, v.z * 2, v.w * 2);
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(mc + 4 * i), "f"(w.x), "f"(w.y), "f"(w.z), "f"(w.w) : "memory");
}

int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  int mcs = -1, fab = -1, posix = -1;
  CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  cuDeviceGetAttribute(&posix, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev);
  cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  printf("multicast_supported=%d posix_fd=%d fabric=%d\n", mcs, posix, fab);
  CUcontext ctx;
  CK(cuDevicePrimaryCtxRetain(&ctx, dev));
  CK(cuCtxSetCurrent(ctx));
  const size_t want = 8 << 20;
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CK(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t size = (want + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle h;
  CK(cuMemCreate(&h, size, &prop, 0));
  int fd = -1;
  CK(cuMemExportToShareableHandle(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  printf("cuMem gran=%zu size=%zu fd=%d\n", gran, size, fd);
  CUdeviceptr uc;
  CK(cuMemAddressReserve(&uc, size, 0, 0, 0));
  CK(cuMemMap(uc, size, 0, h, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, size, &acc, 1));
  if (mcs != 1) { printf("no multicast: done\n"); return 0; }
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.size = size;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t mgran = 0, mmin = 0;
  CK(cuMulticastGetGranularity(&mgran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CK(cuMulticastGetGranularity(&mmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  printf("mc gran recommended=%zu minimum=%zu\n", mgran, mmin);
  if (size % mmin) { printf("size not a multiple of the multicast minimum granularity\n"); return 1; }
  CUmemGenericAllocationHandle mh;
  CUresult cr = cuMulticastCreate(&mh, &mp);
  printf("cuMulticastCreate(posix fd) -> %d\n", int(cr));
  if (cr != CUDA_SUCCESS) {
    mp.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
    cr = cuMulticastCreate(&mh, &mp);
    printf("cuMulticastCreate(fabric) -> %d\n", int(cr));
  }
  if (cr != CUDA_SUCCESS) {
    mp.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
    cr = cuMulticastCreate(&mh, &mp);
    printf("cuMulticastCreate(none) -> %d\n", int(cr));
  }
  if (cr != CUDA_SUCCESS) {
    mp.numDevices = 2; mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    cr = cuMulticastCreate(&mh, &mp);
    printf("cuMulticastCreate(2 devices, posix) -> %d\n", int(cr));
    int ndev = 0; cuDeviceGetCount(&ndev); printf("visible devices %d\n", ndev);
    return 1;
  }
  CK(cuMulticastAddDevice(mh, dev));
  CK(cuMulticastBindMem(mh, 0, h, 0, size, 0));
  CUdeviceptr mc;
  CK(cuMemAddressReserve(&mc, size, mgran, 0, 0));
  CK(cuMemMap(mc, size, 0, mh, 0));
  CK(cuMemSetAccess(mc, size, &acc, 1));
  const int n = 1 << 20;
  float* hbuf = new float[n];
  for (int i = 0; i < n; ++i) hbuf[i] = float(i % 1000) * 0.5f;
  CK(cuMemcpyHtoD(uc, hbuf, n * 4));
  CUdeviceptr out;
  CK(cuMemAlloc(&out, n * 4));
  mm_kernel<<<n / 4 / 256, 256>>>((float*)mc, (float*)uc, (float*)out, n);
  CK(cuCtxSynchronize());
  float* o = new float[n];
  float* u2 = new float[n];
  CK(cuMemcpyDtoH(o, out, n * 4));
  CK(cuMemcpyDtoH(u2, uc, n * 4));
  int bad = 0;
  for (int i = 0; i < n; ++i) bad += (o[i] != hbuf[i]) + (u2[i] != 2 * hbuf[i]);
  printf("multimem ld_reduce/st over a 1-device multicast object: %s (bad=%d)\n", bad ? "WRONG" : "ok", bad);
  return 0;
}
