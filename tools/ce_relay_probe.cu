// Copy-engine relay chain over NVLink (diagnostics; one process, G GPUs).
// GPU 0 holds a `total`-byte source; GPU k (k >= 1) receives it into its
// leader buffer from GPU k-1, piece by piece, and forwards each piece to GPU
// k+1 once it has landed — the library's copy-engine relay (ce_transport=3)
// without its in-host fan-out. Which part of the chain costs time?
//   flags       each forward waits for the piece's flag (cuStreamWaitValue32
//               GEQ), each copy raises the next GPU's flag after it
//               (cuStreamWriteValue32, default = with a memory barrier)
//   (flag writes without the memory barrier are refused on this driver:
//   CU_STREAM_WRITE_VALUE_NO_MEMORY_BARRIER -> CUDA_ERROR_INVALID_VALUE)
//   nowait      forwards issued without waiting (timing only: the bytes
//               forwarded are stale) — the chain's pure transfer time
//   events      waits as cross-device cudaStreamWaitEvent instead of flags
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/ce_relay_probe tools/ce_relay_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) {                                                                \
      std::printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                         \
    }                                                                                       \
  } while (0)
#define CU(x)                                                    \
  do {                                                           \
    CUresult r_ = (x);                                           \
    if (r_ != CUDA_SUCCESS) {                                    \
      std::printf("FAIL %s:%d %s -> %d\n", __FILE__, __LINE__, #x, (int)r_); \
      std::exit(1);                                              \
    }                                                            \
  } while (0)

int G = 4;
std::vector<char*> buf;         // GPU 0: source; others: leader
std::vector<uint32_t*> flags;   // per GPU: one slot per piece
std::vector<cudaStream_t> st;
std::vector<cudaEvent_t> t0, t1;
uint32_t epoch = 0;

enum Mode { kFlags, kFlagsNoMb, kNoWait, kEvents };

// GPU 0's local work in the library's relay phase: the source copied to its
// two local replicas by SMs (read once, two stores), concurrently with the
// chain's first hop. ctas = 0: no local work.
__global__ void local_fanout(const int4* __restrict__ src, int4* __restrict__ a, int4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const int4 v = src[i];
    a[i] = v;
    b[i] = v;
  }
}
// The forwarders' in-host fan-out: every CTA waits for piece p's flag, then
// copies its share of the piece from the leader into the second replica.
__global__ void hop_fanout(const uint32_t* flags, uint32_t epoch, const int4* __restrict__ leader,
                           int4* __restrict__ rep, size_t piece16, size_t n16) {
  const size_t P = (n16 + piece16 - 1) / piece16;
  for (size_t p = 0; p < P; ++p) {
    if (threadIdx.x == 0) {
      uint32_t v;
      do {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + p) : "memory");
        if (v < epoch) __nanosleep(256);
      } while (v < epoch);
    }
    __syncthreads();
    const size_t lo = p * piece16, hi = lo + piece16 < n16 ? lo + piece16 : n16;
    for (size_t i = lo + blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < hi; i += size_t(gridDim.x) * blockDim.x)
      rep[i] = leader[i];
  }
}
int g_hop_ctas = 0;
std::vector<char*> g_hop_rep;
std::vector<cudaStream_t> g_hop_stream;
int g_local_ctas = 0;
char* g_rep[2] = {nullptr, nullptr};
cudaStream_t g_local_stream = nullptr;

double run(Mode mode, size_t total, size_t piece, int reps = 3) {
  const int P = static_cast<int>((total + piece - 1) / piece);
  std::vector<std::vector<cudaEvent_t>> arrived(G, std::vector<cudaEvent_t>(P));
  if (mode == kEvents)
    for (int g = 1; g < G; ++g) {  // recorded by GPU g-1's stream: created on that device
      CK(cudaSetDevice(g - 1));
      for (int p = 0; p < P; ++p) CK(cudaEventCreateWithFlags(&arrived[g][p], cudaEventDisableTiming));
    }
  double best = 1e30;
  for (int r = 0; r < reps + 1; ++r) {
    ++epoch;
    for (int g = 0; g < G; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaDeviceSynchronize());
    }
    CK(cudaSetDevice(0));
    CK(cudaEventRecord(t0[0], st[0]));
    for (int g = 1; g < G; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaStreamWaitEvent(st[g], t0[0], 0));  // every stream starts with GPU 0's
    }
    if (g_local_ctas > 0) {
      CK(cudaSetDevice(0));
      CK(cudaStreamWaitEvent(g_local_stream, t0[0], 0));
      local_fanout<<<g_local_ctas, 512, 0, g_local_stream>>>(reinterpret_cast<const int4*>(buf[0]),
                                                              reinterpret_cast<int4*>(g_rep[0]),
                                                              reinterpret_cast<int4*>(g_rep[1]), total / 16);
      CK(cudaGetLastError());
    }
    if (g_hop_ctas > 0)
      for (int g = 1; g < G; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaStreamWaitEvent(g_hop_stream[g], t0[0], 0));
        hop_fanout<<<g_hop_ctas, 512, 0, g_hop_stream[g]>>>(flags[g], epoch, reinterpret_cast<const int4*>(buf[g]),
                                                            reinterpret_cast<int4*>(g_hop_rep[g]), piece / 16, total / 16);
        CK(cudaGetLastError());
      }
    // issue per GPU in piece order (the host issues GPU by GPU; the streams run concurrently)
    for (int g = 0; g + 1 < G; ++g) {
      CK(cudaSetDevice(g));
      for (int p = 0; p < P; ++p) {
        const size_t off = static_cast<size_t>(p) * piece, w = std::min(piece, total - off);
        if (g > 0) {
          if (mode == kFlags || mode == kFlagsNoMb)
            CU(cuStreamWaitValue32(st[g], (CUdeviceptr)(flags[g] + p), epoch, CU_STREAM_WAIT_VALUE_GEQ));
          else if (mode == kEvents)
            CK(cudaStreamWaitEvent(st[g], arrived[g][p], 0));
        }
        CK(cudaMemcpyAsync(buf[g + 1] + off, buf[g] + off, w, cudaMemcpyDeviceToDevice, st[g]));
        if (mode == kFlags)
          CU(cuStreamWriteValue32(st[g], (CUdeviceptr)(flags[g + 1] + p), epoch, CU_STREAM_WRITE_VALUE_DEFAULT));
        else if (mode == kFlagsNoMb)
          CU(cuStreamWriteValue32(st[g], (CUdeviceptr)(flags[g + 1] + p), epoch,
                                  CU_STREAM_WRITE_VALUE_NO_MEMORY_BARRIER));
        else if (mode == kEvents)
          CK(cudaEventRecord(arrived[g + 1][p], st[g]));
      }
    }
    // the chain's time: GPU 0's start to the last forwarder's end, on GPU 0's clock
    for (int g = 1; g < G; ++g) {
      CK(cudaSetDevice(g));
      if (g_hop_ctas > 0) {  // the hop's end includes its fan-out
        CK(cudaEventRecord(t1[g], g_hop_stream[g]));
        CK(cudaStreamWaitEvent(st[g], t1[g], 0));
      }
      CK(cudaEventRecord(t1[g], st[g]));
    }
    CK(cudaSetDevice(0));
    for (int g = 1; g < G; ++g) CK(cudaStreamWaitEvent(st[0], t1[g], 0));
    if (g_local_ctas > 0) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CK(cudaEventRecord(e, g_local_stream));
      CK(cudaStreamWaitEvent(st[0], e, 0));
      CK(cudaEventDestroy(e));
    }
    CK(cudaEventRecord(t1[0], st[0]));
    CK(cudaEventSynchronize(t1[0]));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, t0[0], t1[0]));
    if (r > 0 && ms < best) best = ms;
  }
  if (mode == kEvents)
    for (int g = 1; g < G; ++g) {
      CK(cudaSetDevice(g - 1));
      for (int p = 0; p < P; ++p) CK(cudaEventDestroy(arrived[g][p]));
    }
  return best;
}

int main(int argc, char** argv) {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  G = n;
  if (G < 3) {
    std::printf("needs >= 3 GPUs\n");
    return 1;
  }
  const size_t total = size_t(16) << 30;
  buf.resize(G);
  flags.resize(G);
  st.resize(G);
  t0.resize(G);
  t1.resize(G);
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < G; ++h)
      if (h != g) CK(cudaDeviceEnablePeerAccess(h, 0));
    CK(cudaMalloc(&buf[g], total));
    CK(cudaMemset(buf[g], g, total));
    CK(cudaMalloc(&flags[g], 1 << 20));
    CK(cudaMemset(flags[g], 0, 1 << 20));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&t0[g]));
    CK(cudaEventCreate(&t1[g]));  // (only GPU 0's pair is timed; the others order streams)
  }
  std::printf("chain 0 -> ... -> %d, %zu GiB\n", G - 1, total >> 30);
  const char* names[] = {"flags", "flags/nomb", "nowait", "events"};
  if (argc > 2 && std::string(argv[1]) == "hop") {  // forwarders' fan-out kernels at these CTA counts
    g_hop_rep.assign(G, nullptr);
    g_hop_stream.assign(G, nullptr);
    for (int g = 1; g < G; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaMalloc(&g_hop_rep[g], total));
      CK(cudaStreamCreateWithFlags(&g_hop_stream[g], cudaStreamNonBlocking));
    }
    for (int a = 2; a < argc; ++a) {
      g_hop_ctas = std::atoi(argv[a]);
      for (size_t piece_mib : {192, 256}) {
        const double ms = run(kFlags, total, piece_mib << 20);
        std::printf("flags + hop fan-out ctas=%4d  piece %4zu MiB  %8.3f ms  %7.1f GB/s per link\n", g_hop_ctas,
                    piece_mib, ms, total / (ms * 1e-3) / 1e9);
        std::fflush(stdout);
      }
    }
    return 0;
  }
  if (argc > 1) {  // with GPU 0's local fan-out (source -> two local replicas by SMs) at these CTA counts
    CK(cudaSetDevice(0));
    CK(cudaMalloc(&g_rep[0], total));
    CK(cudaMalloc(&g_rep[1], total));
    CK(cudaStreamCreateWithFlags(&g_local_stream, cudaStreamNonBlocking));
    for (int a = 1; a < argc; ++a) {
      g_local_ctas = std::atoi(argv[a]);
      for (size_t piece_mib : {192, 256}) {
        const double ms = run(kFlags, total, piece_mib << 20);
        std::printf("flags + GPU0 local fan-out ctas=%4d  piece %4zu MiB  %8.3f ms  %7.1f GB/s per link\n", g_local_ctas,
                    piece_mib, ms, total / (ms * 1e-3) / 1e9);
        std::fflush(stdout);
      }
    }
    return 0;
  }
  for (size_t piece_mib : {64, 256, 1024}) {
    for (Mode m : {kFlags, kNoWait, kEvents}) {
      const double ms = run(m, total, piece_mib << 20);
      std::printf("%-11s piece %5zu MiB  %8.3f ms  %7.1f GB/s per link\n", names[m], piece_mib, ms,
                  total / (ms * 1e-3) / 1e9);
      std::fflush(stdout);
    }
  }
  return 0;
}
