// NVLink store-path probe (diagnostics; one process, GPUs 0 and 1).
// What limits an SM-driven peer push? Copies `bytes` from a local buffer to
// the peer GPU's buffer with several store flavours, one direction (uni) and
// both directions at once (bi, the all-gather case), beside the copy engine:
//   v4      16-byte ld.global.nc + st.global per thread
//   v4cs    the same with st.global.cs (streaming, evict-first)
//   v8      32-byte (256-bit) ld/st per thread (sm_100)
//   bulk    TMA: cp.async.bulk global->shared, shared->global (16 KiB stages)
//   ce      cudaMemcpyPeerAsync (copy engine); ce/<MiB> the same as 1D copies
//           of that size, ce2d/<KiB> strided rows (pitch 8x), ce+hbm the CE
//           push beside a local SM copy kernel of the same size
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/nvlink_probe tools/nvlink_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

__global__ void k_v4(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(src + i);
    dst[i] = v;
  }
}

__global__ void k_v4cs(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(src + i);
    __stcs(dst + i, v);
  }
}

__global__ void k_v8(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  // n counts 16-byte units; each thread moves 32 bytes
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; 2 * i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t r[8];
    const void* s = src + 2 * i;
    void* d = dst + 2 * i;
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "l"(s));
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(d), "r"(r[0]), "r"(r[1]), "r"(r[2]),
                 "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
  }
}

constexpr int kStage = 16384, kStages = 4;

__global__ void k_bulk(const char* __restrict__ src, char* __restrict__ dst, size_t bytes) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[kStages];
  const size_t chunks = bytes / kStage;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase[kStages] = {0, 0, 0, 0};
  size_t first = blockIdx.x;
  // prologue: issue up to kStages loads
  int inflight = 0;
  size_t c = first;
  for (int s = 0; s < kStages && c < chunks; ++s, c += gridDim.x, ++inflight) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t sm = (uint32_t)__cvta_generic_to_shared(smem + s * kStage);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(kStage));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sm),
                 "l"(src + c * kStage), "r"(kStage), "r"(a)
                 : "memory");
  }
  size_t out = first;
  int s = 0;
  while (out < chunks) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t sm = (uint32_t)__cvta_generic_to_shared(smem + s * kStage);
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(a),
        "r"(phase[s]));
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + out * kStage), "r"(sm),
                 "r"(kStage)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (c < chunks) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(kStage));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sm),
                   "l"(src + c * kStage), "r"(kStage), "r"(a)
                   : "memory");
      c += gridDim.x;
    }
    out += gridDim.x;
    s = (s + 1) % kStages;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static cudaStream_t st2[2];  // second stream per GPU (ce+hbm)
constexpr int kSx = 8;
static cudaStream_t sx[2][kSx];  // CE fan-out streams
static cudaEvent_t jx[2][kSx];

static int run(const char* name, int dirs, size_t bytes, char** src, char** dst, cudaStream_t* st, int ctas,
               int threads) {
  cudaEvent_t e0[2], e1[2], j[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaEventCreateWithFlags(&j[d], cudaEventDisableTiming));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  // gce/<MiB>: the ce/<MiB> copies captured once in a CUDA graph
  cudaGraphExec_t gx[2] = {nullptr, nullptr};
  if (!std::strncmp(name, "gce/", 4)) {
    const size_t chunk = size_t(std::atoi(name + 4)) << 20;
    for (int d = 0; d < dirs; ++d) {
      CK(cudaSetDevice(d));
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(st[d], cudaStreamCaptureModeThreadLocal));
      for (size_t off = 0; off < bytes; off += chunk)
        CK(cudaMemcpyAsync(dst[1 - d] + off, src[d] + off, chunk < bytes - off ? chunk : bytes - off,
                           cudaMemcpyDefault, st[d]));
      CK(cudaStreamEndCapture(st[d], &g));
      CK(cudaGraphInstantiate(&gx[d], g, 0));
      CK(cudaGraphDestroy(g));
    }
  }
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaDeviceSynchronize());
    }
    for (int d = 0; d < dirs; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaEventRecord(e0[d], st[d]));
      CK(cudaStreamWaitEvent(st2[d], e0[d], 0));
      for (int k = 0; k < kSx; ++k) CK(cudaStreamWaitEvent(sx[d][k], e0[d], 0));
      char* to = dst[1 - d];
      const size_t n16 = bytes / 16;
      if (!std::strcmp(name, "v4"))
        k_v4<<<ctas, threads, 0, st[d]>>>((const uint4*)src[d], (uint4*)to, n16);
      else if (!std::strcmp(name, "v4cs"))
        k_v4cs<<<ctas, threads, 0, st[d]>>>((const uint4*)src[d], (uint4*)to, n16);
      else if (!std::strcmp(name, "v8"))
        k_v8<<<ctas, threads, 0, st[d]>>>((const uint4*)src[d], (uint4*)to, n16);
      else if (!std::strcmp(name, "bulk"))
        k_bulk<<<ctas, 32, kStages * kStage, st[d]>>>(src[d], to, bytes);
      else if (gx[d])
        CK(cudaGraphLaunch(gx[d], st[d]));
      else if (!std::strncmp(name, "ce/", 3)) {  // ce/<chunk MiB>[x<streams>]: 1D copies of that size
        const size_t chunk = size_t(std::atoi(name + 3)) << 20;
        const char* x = std::strchr(name, 'x');
        const int ns = x ? std::atoi(x + 1) : 1;
        int i = 0;
        for (size_t off = 0; off < bytes; off += chunk, ++i) {
          cudaStream_t s = ns == 1 ? st[d] : sx[d][i % ns];
          CK(cudaMemcpyAsync(to + off, src[d] + off, chunk < bytes - off ? chunk : bytes - off, cudaMemcpyDefault, s));
        }
        for (int k = 0; k < ns && ns > 1; ++k) {
          CK(cudaEventRecord(jx[d][k], sx[d][k]));
          CK(cudaStreamWaitEvent(st[d], jx[d][k], 0));
        }
      } else if (!std::strncmp(name, "ce2d/", 5)) {  // ce2d/<row KiB>: rows into a 8x pitch
        const size_t w = size_t(std::atoi(name + 5)) << 10, pitch = 8 * w, rows = bytes / pitch;
        CK(cudaMemcpy2DAsync(to, pitch, src[d], w, w, rows, cudaMemcpyDefault, st[d]));
      } else if (!std::strcmp(name, "ce+hbm")) {  // CE push beside a local SM copy of the same size
        CK(cudaMemcpyAsync(to, src[d], bytes, cudaMemcpyDefault, st[d]));
        k_v4<<<ctas, 512, 0, st2[d]>>>((const uint4*)(src[d]), (uint4*)(dst[d]), bytes / 16);
      } else
        CK(cudaMemcpyPeerAsync(to, 1 - d, src[d], d, bytes, st[d]));
      CK(cudaGetLastError());
      CK(cudaEventRecord(j[d], st2[d]));
      CK(cudaStreamWaitEvent(st[d], j[d], 0));
      CK(cudaEventRecord(e1[d], st[d]));
    }
    float ms = 0;
    for (int d = 0; d < dirs; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaEventSynchronize(e1[d]));
      float m = 0;
      CK(cudaEventElapsedTime(&m, e0[d], e1[d]));
      if (m > ms) ms = m;
    }
    if (rep > 0 && ms < best) best = ms;
  }
  std::printf("%-5s %-3s ctas=%-4d thr=%-4d %8.1f GB/s per direction\n", name, dirs == 2 ? "bi" : "uni", ctas, threads,
              (std::strncmp(name, "ce2d/", 5) ? bytes : bytes / 8) / (best * 1e6));
  return 0;
}

int main() {
  const size_t bytes = size_t(2) << 30;
  char *src[2], *dst[2];
  cudaStream_t st[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&src[d], bytes));
    CK(cudaMalloc(&dst[d], bytes));
    CK(cudaMemset(src[d], d + 1, bytes));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&st2[d], cudaStreamNonBlocking));
    for (int k = 0; k < kSx; ++k) {
      CK(cudaStreamCreateWithFlags(&sx[d][k], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&jx[d][k], cudaEventDisableTiming));
    }
    CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kStage));
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int dirs = 1; dirs <= 2; ++dirs) {
    for (const char* k : {"ce", "ce/1", "ce/4", "ce/16", "ce/64", "ce/256", "ce2d/1", "ce2d/4", "ce/1x4",
                          "ce/4x4", "gce/1", "gce/4", "gce/16", "gce/64"})
      if (run(k, dirs, bytes, src, dst, st, 0, 0)) return 1;
    if (run("ce+hbm", dirs, bytes, src, dst, st, sms * 2, 0)) return 1;
    for (int mult : {1, 2, 4})
      for (const char* k : {"v4", "v4cs", "v8"})
        if (run(k, dirs, bytes, src, dst, st, sms * mult, 512)) return 1;
    for (int mult : {1, 2, 3})
      if (run("bulk", dirs, bytes, src, dst, st, sms * mult, 32)) return 1;
    for (int c : {16, 32, 64})
      if (run("v4", dirs, bytes, src, dst, st, c, 1024)) return 1;
  }
  // verify the last copy direction 1 -> 0 content
  CK(cudaSetDevice(0));
  unsigned char h = 0;
  CK(cudaMemcpy(&h, dst[0] + bytes - 1, 1, cudaMemcpyDeviceToHost));
  std::printf("check %s\n", h == 2 ? "ok" : "BAD");
  return 0;
}
