// Standalone NVLS multicast probe (diagnostics; single process, all GPUs).
// Build: nvcc -o tools/mc_probe tools/mc_probe.cu -L/usr/local/cuda/lib64/stubs -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

#define CK(x)                                                       \
  do {                                                              \
    CUresult r_ = (x);                                              \
    if (r_ != CUDA_SUCCESS) {                                       \
      const char* s_ = nullptr;                                     \
      cuGetErrorString(r_, &s_);                                    \
      std::printf("FAIL %s -> %d %s\n", #x, (int)r_, s_ ? s_ : ""); \
      return 1;                                                     \
    }                                                               \
  } while (0)

static int attempt(int ndev, size_t want, int handle_types, int phys_handle, int gdr) {
  CUmulticastObjectProp mp;
  std::memset(&mp, 0, sizeof(mp));
  mp.numDevices = ndev;
  mp.size = want;
  mp.handleTypes = handle_types;
  size_t mgmin = 0, mgrec = 0;
  CK(cuMulticastGetGranularity(&mgmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CK(cuMulticastGetGranularity(&mgrec, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CUmemAllocationProp ap;
  std::memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = (CUmemAllocationHandleType)phys_handle;
  ap.allocFlags.gpuDirectRDMACapable = gdr;
  size_t agmin = 0, agrec = 0;
  CK(cuMemGetAllocationGranularity(&agmin, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  CK(cuMemGetAllocationGranularity(&agrec, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  size_t g = mgrec > agrec ? mgrec : agrec;
  size_t size = (want + g - 1) / g * g;
  std::printf("ndev=%d handles=%d phys=%d gdr=%d mc_gran min=%zu rec=%zu alloc_gran min=%zu rec=%zu size=%zu\n",
              ndev, handle_types, phys_handle, gdr, mgmin, mgrec, agmin, agrec, size);
  mp.size = size;
  CUmemGenericAllocationHandle mc;
  CK(cuMulticastCreate(&mc, &mp));
  for (int d = 0; d < ndev; ++d) CK(cuMulticastAddDevice(mc, d));
  for (int d = 0; d < ndev; ++d) {
    cudaSetDevice(d);
    ap.location.id = d;
    CUmemGenericAllocationHandle mem;
    CK(cuMemCreate(&mem, size, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, mem, 0, size, 0));
    std::printf("  bound device %d\n", d);
  }
  std::printf("  OK\n");
  return 0;
}

int main() {
  CK(cuInit(0));
  int n = 0;
  cudaGetDeviceCount(&n);
  for (int d = 0; d < n; ++d) {
    cudaSetDevice(d);
    cudaFree(nullptr);
  }
  int sup = 0;
  CK(cuDeviceGetAttribute(&sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, 0));
  std::printf("devices %d multicast %d\n", n, sup);
  const size_t want = size_t(64) << 20;
  attempt(n, want, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0, 0);
  attempt(n, want, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  attempt(n, want, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 1);
  attempt(n, want, 0, 0, 0);
  return 0;
}
