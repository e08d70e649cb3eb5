// NVLS multicast objects for the one-to-many replica broadcast (K3).
//
// A multicast object spans one buffer per participating GPU. A store through
// its multicast address (multimem.st) leaves the writing GPU once and is
// replicated by the NVSwitch into every member's memory — the egress of a
// broadcast to k replicas drops from k copies to one. The driver API is
// resolved at run time (cudaGetDriverEntryPoint), so the library has no link
// dependency on libcuda and still loads on a CPU-only host.
//
// Protocol for one process per GPU (see runtime.py::Multicast):
//   root:   rr_mcast_create  -> POSIX fd (shared to peers over SCM_RIGHTS)
//   others: rr_mcast_import(fd)
//   all:    (barrier: every device added)  rr_mcast_bind -> unicast + multicast VA
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <cstring>
#include <memory>
#include <string>

#include "rr_internal.hpp"
#include "rr_realloc.h"

namespace {


struct Driver {
  bool ok = false;
  decltype(&cuMulticastCreate) mcCreate = nullptr;
  decltype(&cuMulticastAddDevice) mcAddDevice = nullptr;
  decltype(&cuMulticastBindMem) mcBindMem = nullptr;
  decltype(&cuMulticastUnbind) mcUnbind = nullptr;
  decltype(&cuMulticastGetGranularity) mcGranularity = nullptr;
  decltype(&cuMemCreate) memCreate = nullptr;
  decltype(&cuMemRelease) memRelease = nullptr;
  decltype(&cuMemMap) memMap = nullptr;
  decltype(&cuMemUnmap) memUnmap = nullptr;
  decltype(&cuMemAddressReserve) addrReserve = nullptr;
  decltype(&cuMemAddressFree) addrFree = nullptr;
  decltype(&cuMemSetAccess) setAccess = nullptr;
  decltype(&cuMemExportToShareableHandle) exportHandle = nullptr;
  decltype(&cuMemImportFromShareableHandle) importHandle = nullptr;
  decltype(&cuMemGetAllocationGranularity) allocGranularity = nullptr;
  decltype(&cuDeviceGetAttribute) devAttr = nullptr;
  decltype(&cuGetErrorString) errString = nullptr;
};

template <class F>
bool resolve(const char* name, F& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      !p) {
    cudaGetLastError();
    return false;
  }
  fn = reinterpret_cast<F>(p);
  return true;
}

const Driver& driver() {
  static Driver d = [] {
    Driver x;
    x.ok = resolve("cuMulticastCreate", x.mcCreate) && resolve("cuMulticastAddDevice", x.mcAddDevice) &&
           resolve("cuMulticastBindMem", x.mcBindMem) && resolve("cuMulticastUnbind", x.mcUnbind) &&
           resolve("cuMulticastGetGranularity", x.mcGranularity) && resolve("cuMemCreate", x.memCreate) &&
           resolve("cuMemRelease", x.memRelease) && resolve("cuMemMap", x.memMap) &&
           resolve("cuMemUnmap", x.memUnmap) && resolve("cuMemAddressReserve", x.addrReserve) &&
           resolve("cuMemAddressFree", x.addrFree) && resolve("cuMemSetAccess", x.setAccess) &&
           resolve("cuMemExportToShareableHandle", x.exportHandle) &&
           resolve("cuMemImportFromShareableHandle", x.importHandle) &&
           resolve("cuMemGetAllocationGranularity", x.allocGranularity) &&
           resolve("cuDeviceGetAttribute", x.devAttr) && resolve("cuGetErrorString", x.errString);
    return x;
  }();
  return d;
}

struct Fail {
  rr_status status;
  std::string msg;
};

void cu(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* s = nullptr;
  if (driver().errString) driver().errString(r, &s);
  throw Fail{RR_ECUDA, std::string(what) + ": " + (s ? s : "CUDA driver error")};
}

template <class F>
rr_status run(F&& f) {
  try {
    f();
    return RR_OK;
  } catch (const Fail& e) {
    rr::set_last_error(e.msg);
    return e.status;
  }
}

size_t round_up(size_t v, size_t g) { return (v + g - 1) / g * g; }

}  // namespace

struct rr_mcast {
  int cuda_device = 0;
  int n_devices = 0;
  size_t size = 0;
  CUmemGenericAllocationHandle mc = 0;
  CUmemGenericAllocationHandle mem = 0;
  CUdeviceptr uc_va = 0, mc_va = 0;
  bool bound = false;
  int fd = -1;

  rr_mcast() = default;
  rr_mcast(const rr_mcast&) = delete;
  rr_mcast& operator=(const rr_mcast&) = delete;
  ~rr_mcast();  // releases whatever exists, also after a failed create/import/bind
};

rr_status rr_mcast_supported(int cuda_device, int* supported) {
  return run([&] {
    *supported = 0;
    if (!driver().ok) return;
    int v = 0;
    if (cudaSetDevice(cuda_device) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    cu(driver().devAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cuda_device), "cuDeviceGetAttribute");
    *supported = v;
  });
}

static void init_common(rr_mcast* m, int cuda_device, size_t bytes, int n_devices) {
  if (!driver().ok) throw Fail{RR_EUNSUPPORTED, "CUDA driver lacks the multicast API"};
  if (cudaSetDevice(cuda_device) != cudaSuccess) {
    cudaGetLastError();
    throw Fail{RR_ECUDA, "cudaSetDevice failed"};
  }
  cudaFree(nullptr);  // make sure the primary context exists
  int sup = 0;
  cu(driver().devAttr(&sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cuda_device), "cuDeviceGetAttribute");
  if (!sup) throw Fail{RR_EUNSUPPORTED, "device does not support NVLS multicast"};
  CUmulticastObjectProp prop;
  std::memset(&prop, 0, sizeof(prop));
  prop.numDevices = static_cast<unsigned>(n_devices);
  prop.size = bytes;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g = 0;
  cu(driver().mcGranularity(&g, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
  m->cuda_device = cuda_device;
  m->n_devices = n_devices;
  m->size = round_up(bytes, g);
}

rr_status rr_mcast_create(int cuda_device, size_t bytes, int n_devices, int* fd_out, size_t* size_out,
                          rr_mcast** out) {
  auto m = std::make_unique<rr_mcast>();
  const rr_status st = run([&] {
    if (n_devices < 1 || !fd_out || !size_out || !out) throw Fail{RR_EINVAL, "bad multicast arguments"};
    init_common(m.get(), cuda_device, bytes, n_devices);
    CUmulticastObjectProp prop;
    std::memset(&prop, 0, sizeof(prop));
    prop.numDevices = static_cast<unsigned>(n_devices);
    prop.size = m->size;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    cu(driver().mcCreate(&m->mc, &prop), "cuMulticastCreate");
    int fd = -1;
    cu(driver().exportHandle(&fd, m->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
       "cuMemExportToShareableHandle");
    m->fd = fd;
    cu(driver().mcAddDevice(m->mc, cuda_device), "cuMulticastAddDevice");
    *fd_out = fd;
    *size_out = m->size;
  });
  if (st == RR_OK) *out = m.release();
  return st;
}

rr_status rr_mcast_import(int cuda_device, int fd, size_t size, int n_devices, rr_mcast** out) {
  auto m = std::make_unique<rr_mcast>();
  const rr_status st = run([&] {
    if (!out || fd < 0) throw Fail{RR_EINVAL, "bad multicast arguments"};
    init_common(m.get(), cuda_device, size, n_devices);
    m->size = size;
    cu(driver().importHandle(&m->mc, reinterpret_cast<void*>(static_cast<intptr_t>(fd)),
                             CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
       "cuMemImportFromShareableHandle");
    cu(driver().mcAddDevice(m->mc, cuda_device), "cuMulticastAddDevice");
  });
  if (st == RR_OK) *out = m.release();
  return st;
}

rr_status rr_mcast_bind(rr_mcast* m, void** unicast_ptr, void** multicast_ptr) {
  return run([&] {
    if (!m || !unicast_ptr || !multicast_ptr) throw Fail{RR_EINVAL, "bad multicast arguments"};
    if (cudaSetDevice(m->cuda_device) != cudaSuccess) {
      cudaGetLastError();
      throw Fail{RR_ECUDA, "cudaSetDevice failed"};
    }
    CUmemAllocationProp prop;
    std::memset(&prop, 0, sizeof(prop));
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = m->cuda_device;
    // Binding requires the member memory to carry the multicast object's
    // handle type (tools/mc_probe.cu: without it cuMulticastBindMem fails).
    prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    cu(driver().memCreate(&m->mem, m->size, &prop, 0), "cuMemCreate");
    cu(driver().mcBindMem(m->mc, 0, m->mem, 0, m->size, 0), "cuMulticastBindMem");
    m->bound = true;
    CUmemAccessDesc acc;
    std::memset(&acc, 0, sizeof(acc));
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = m->cuda_device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    size_t g = 0;
    cu(driver().allocGranularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
    const size_t align = g > (size_t{2} << 20) ? g : (size_t{2} << 20);
    cu(driver().addrReserve(&m->uc_va, m->size, align, 0, 0), "cuMemAddressReserve(unicast)");
    cu(driver().memMap(m->uc_va, m->size, 0, m->mem, 0), "cuMemMap(unicast)");
    cu(driver().setAccess(m->uc_va, m->size, &acc, 1), "cuMemSetAccess(unicast)");
    cu(driver().addrReserve(&m->mc_va, m->size, align, 0, 0), "cuMemAddressReserve(multicast)");
    cu(driver().memMap(m->mc_va, m->size, 0, m->mc, 0), "cuMemMap(multicast)");
    cu(driver().setAccess(m->mc_va, m->size, &acc, 1), "cuMemSetAccess(multicast)");
    *unicast_ptr = reinterpret_cast<void*>(m->uc_va);
    *multicast_ptr = reinterpret_cast<void*>(m->mc_va);
  });
}

rr_status rr_mcast_size(const rr_mcast* m, size_t* size) {
  return run([&] {
    if (!m || !size) throw Fail{RR_EINVAL, "bad multicast arguments"};
    *size = m->size;
  });
}

rr_mcast::~rr_mcast() {
  const Driver& d = driver();
  if (d.ok && (mc || mem || uc_va || mc_va)) {
    cudaSetDevice(cuda_device);
    cudaDeviceSynchronize();
    if (mc_va) {
      d.memUnmap(mc_va, size);
      d.addrFree(mc_va, size);
    }
    if (uc_va) {
      d.memUnmap(uc_va, size);
      d.addrFree(uc_va, size);
    }
    if (bound) d.mcUnbind(mc, cuda_device, 0, size);
    if (mem) d.memRelease(mem);
    if (mc) d.memRelease(mc);
  }
  if (fd >= 0) close(fd);
}

void rr_mcast_destroy(rr_mcast* m) { delete m; }

// ---- a member's memory reached by the other GPUs with ordinary peer
// stores (the schemes that do not use the multicast address): the member's
// physical allocation is exported as a POSIX fd and mapped by each peer ----

rr_status rr_mcast_export_member(rr_mcast* m, int* fd_out) {
  return run([&] {
    if (!m || !fd_out || !m->mem) throw Fail{RR_EINVAL, "multicast member not bound"};
    int fd = -1;
    cu(driver().exportHandle(&fd, m->mem, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
       "cuMemExportToShareableHandle(member)");
    *fd_out = fd;
  });
}

struct rr_peer_mem {
  int cuda_device = 0;
  size_t size = 0;
  CUmemGenericAllocationHandle mem = 0;
  CUdeviceptr va = 0;
  bool mapped = false;
  ~rr_peer_mem() {
    const Driver& d = driver();
    if (!d.ok) return;
    cudaSetDevice(cuda_device);
    if (mapped) d.memUnmap(va, size);
    if (va) d.addrFree(va, size);
    if (mem) d.memRelease(mem);
  }
};

rr_status rr_peer_mem_import(int cuda_device, int fd, size_t size, void** ptr, rr_peer_mem** out) {
  auto p = std::make_unique<rr_peer_mem>();
  const rr_status st = run([&] {
    if (!driver().ok) throw Fail{RR_EUNSUPPORTED, "CUDA driver lacks the VMM API"};
    if (fd < 0 || !ptr || !out || size == 0) throw Fail{RR_EINVAL, "bad peer memory arguments"};
    if (cudaSetDevice(cuda_device) != cudaSuccess) {
      cudaGetLastError();
      throw Fail{RR_ECUDA, "cudaSetDevice failed"};
    }
    p->cuda_device = cuda_device;
    p->size = size;
    cu(driver().importHandle(&p->mem, reinterpret_cast<void*>(static_cast<intptr_t>(fd)),
                             CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
       "cuMemImportFromShareableHandle(peer member)");
    cu(driver().addrReserve(&p->va, size, size_t{2} << 20, 0, 0), "cuMemAddressReserve(peer member)");
    cu(driver().memMap(p->va, size, 0, p->mem, 0), "cuMemMap(peer member)");
    p->mapped = true;
    CUmemAccessDesc acc;
    std::memset(&acc, 0, sizeof(acc));
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = cuda_device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    cu(driver().setAccess(p->va, size, &acc, 1), "cuMemSetAccess(peer member)");
    *ptr = reinterpret_cast<void*>(p->va);
  });
  if (st == RR_OK) *out = p.release();
  return st;
}

void rr_peer_mem_close(rr_peer_mem* p) { delete p; }
