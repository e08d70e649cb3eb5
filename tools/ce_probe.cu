// Copy-engine probe (diagnostics; one process, all visible GPUs, 2..8).
// Can the copy engines beat the ~710 GB/s SM-store ceiling on the plan's
// real piece shapes, and what does each submitted copy cost?
//   a2a/sm           every GPU pushes S bytes to every peer with SM stores (v4)
//   a2a/ce<M>[s]     the same with cudaMemcpyAsync pieces of M MiB; s = one
//                    stream per peer (else one stream for all peers)
//   2d/<n>           per peer, n cudaMemcpy2DAsync ops of 4096 rows x 1 KiB
//                    into an 8 KiB pitch (the 7B o_proj tp8 slice shape)
//   mix/<pct>        pct% of each peer's bytes by CE (one stream per peer),
//                    the rest by the SM kernel at the same time
//   h2d/<M>[x<s>]    pinned host -> device, M MiB pieces over s streams
//   rot/ce           all-to-all as G-1 rounds on ONE stream: round r sends the
//                    whole slice to peer (d + r) % G, so every round is a
//                    permutation (each GPU receives from exactly one peer)
//   rot/cepull       the same rounds with each GPU's engine pulling from (d - r) % G
//   pair/sm, pair/ce GPUs paired (d <-> d^1), each pushes 2 GiB to its partner
//                    only (a pipeline-stage remap's pattern): SM stores vs one
//                    whole copy-engine copy
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/ce_probe tools/ce_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
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

constexpr int kMax = 8;
static int G = 0;
static size_t S = size_t(1) << 30;  // bytes per (GPU, peer)
static char* src[kMax];             // G*S: slice p goes to peer p
static char* dst[kMax];             // G*S: slice p comes from peer p
static cudaStream_t st[kMax][kMax + 1];
static cudaEvent_t e0[kMax], e1[kMax], joinev[kMax][kMax + 1];
static int sms = 148;

// Peer-push kernel: CTAs split evenly over the peers, 16 B per thread per iteration.
struct Targets {
  char* to[kMax];
};
__global__ void k_a2a(const char* __restrict__ base, Targets t, int self, int g, size_t s, size_t skip) {
  const int npeer = g - 1;
  const int per = gridDim.x / npeer;
  const int pi = blockIdx.x / per;
  if (pi >= npeer) return;
  const int p = pi < self ? pi : pi + 1;
  const uint4* from = (const uint4*)(base + size_t(p) * s + skip);
  uint4* to = (uint4*)(t.to[p] + size_t(self) * s + skip);
  const size_t n = (s - skip) / 16;
  for (size_t i = (blockIdx.x % per) * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)per * blockDim.x)
    to[i] = __ldg(from + i);
}

__global__ void k_copy(const uint4* __restrict__ from, uint4* __restrict__ to, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    to[i] = __ldg(from + i);
}

static void enqueue_ce(int d, size_t piece, bool per_peer_stream, size_t skip_tail) {
  // copies the first S - skip_tail bytes of each peer slice
  const size_t bytes = S - skip_tail;
  for (int p = 0; p < G; ++p) {
    if (p == d) continue;
    cudaStream_t s = per_peer_stream ? st[d][p] : st[d][kMax];
    char* to = dst[p] + size_t(d) * S;
    const char* from = src[d] + size_t(p) * S;
    for (size_t off = 0; off < bytes; off += piece)
      CK(cudaMemcpyAsync(to + off, from + off, piece < bytes - off ? piece : bytes - off, cudaMemcpyDefault, s));
  }
}

// 2D pieces: rows of 1 KiB from a packed source into an 8 KiB pitch.
static void enqueue_2d(int d, int nops) {
  const size_t w = 1024, rows = 4096, pitch = 8 * w;
  for (int p = 0; p < G; ++p) {
    if (p == d) continue;
    cudaStream_t s = st[d][p];
    char* to = dst[p] + size_t(d) * S;
    const char* from = src[d] + size_t(p) * S;
    for (int k = 0; k < nops; ++k)
      CK(cudaMemcpy2DAsync(to + size_t(k) * rows * pitch, pitch, from + size_t(k) * rows * w, w, w, rows,
                           cudaMemcpyDefault, s));
  }
}

template <class F>
static double timed(F&& enqueue, int reps = 5) {
  double best = 1e30;
  for (int r = 0; r < reps + 1; ++r) {
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaDeviceSynchronize());
    }
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaEventRecord(e0[d], st[d][kMax]));
      for (int p = 0; p < kMax; ++p) CK(cudaStreamWaitEvent(st[d][p], e0[d], 0));
      enqueue(d);
      CK(cudaGetLastError());
      for (int p = 0; p < kMax; ++p) {
        CK(cudaEventRecord(joinev[d][p], st[d][p]));
        CK(cudaStreamWaitEvent(st[d][kMax], joinev[d][p], 0));
      }
      CK(cudaEventRecord(e1[d], st[d][kMax]));
    }
    double ms = 0;
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaEventSynchronize(e1[d]));
      float m = 0;
      CK(cudaEventElapsedTime(&m, e0[d], e1[d]));
      if (m > ms) ms = m;
    }
    if (r > 0 && ms < best) best = ms;
  }
  return best;
}

static void report(const char* name, double bytes_per_gpu, double ms) {
  std::printf("%-14s gpus=%d %10.3f ms %8.1f GB/s per GPU per direction\n", name, G, ms, bytes_per_gpu / (ms * 1e6));
  std::fflush(stdout);
}

int main(int argc, char** argv) {
  CK(cudaGetDeviceCount(&G));
  if (G > kMax) G = kMax;
  if (argc > 1) G = std::atoi(argv[1]);
  if (G < 2) {
    std::printf("need >= 2 GPUs\n");
    return 1;
  }
  S = (size_t(2) << 30) / (G - 1);  // ~2 GiB of egress per GPU
  S &= ~size_t((1 << 20) - 1);
  for (int d = 0; d < G; ++d) {
    CK(cudaSetDevice(d));
    for (int p = 0; p < G; ++p)
      if (p != d) CK(cudaDeviceEnablePeerAccess(p, 0));
    CK(cudaMalloc(&src[d], G * S));
    CK(cudaMalloc(&dst[d], G * S));
    CK(cudaMemset(src[d], d + 1, G * S));
    for (int p = 0; p <= kMax; ++p) {
      CK(cudaStreamCreateWithFlags(&st[d][p], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&joinev[d][p], cudaEventDisableTiming));
    }
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const double egress = double(S) * (G - 1);
  Targets t{};
  for (int p = 0; p < G; ++p) t.to[p] = dst[p];
  const int ctas = (sms * 2 / (G - 1)) * (G - 1);

  {
    // pairwise: d -> d^1 only, 2 GiB (the whole src/dst buffers are >= 2 GiB when G <= 2; else use G*S)
    const size_t pb = std::min(size_t(2) << 30, G * S);
    report("pair/sm", double(pb), timed([&](int d) {
      k_copy<<<sms * 2, 512, 0, st[d][kMax]>>>((const uint4*)src[d], (uint4*)dst[d ^ 1], pb / 16);
    }));
    report("pair/ce", double(pb), timed([&](int d) {
      CK(cudaMemcpyAsync(dst[d ^ 1], src[d], pb, cudaMemcpyDefault, st[d][kMax]));
    }));
    report("pair/ce64", double(pb), timed([&](int d) {
      for (size_t off = 0; off < pb; off += size_t(64) << 20)
        CK(cudaMemcpyAsync(dst[d ^ 1] + off, src[d] + off, std::min(size_t(64) << 20, pb - off), cudaMemcpyDefault,
                           st[d][kMax]));
    }));
  }
  report("rot/ce", egress, timed([&](int d) {
    for (int r = 1; r < G; ++r) {
      const int p = (d + r) % G;
      CK(cudaMemcpyAsync(dst[p] + size_t(d) * S, src[d] + size_t(p) * S, S, cudaMemcpyDefault, st[d][kMax]));
    }
  }));
  report("rot/cepull", egress, timed([&](int d) {  // the same rounds, each GPU's engine pulling from its peer
    for (int r = 1; r < G; ++r) {
      const int p = (d - r + G) % G;
      CK(cudaMemcpyAsync(dst[d] + size_t(p) * S, src[p] + size_t(d) * S, S, cudaMemcpyDefault, st[d][kMax]));
    }
  }));
  report("a2a/sm", egress, timed([&](int d) { k_a2a<<<ctas, 512, 0, st[d][kMax]>>>(src[d], t, d, G, S, 0); }));
  report("a2a/ce-whole", egress, timed([&](int d) { enqueue_ce(d, S, true, 0); }));
  for (int m : {1, 4, 16}) {
    const size_t piece = size_t(m) << 20;
    char nm[32];
    std::snprintf(nm, sizeof nm, "a2a/ce%d", m);
    report(nm, egress, timed([&](int d) { enqueue_ce(d, piece, false, 0); }));
    std::snprintf(nm, sizeof nm, "a2a/ce%ds", m);
    report(nm, egress, timed([&](int d) { enqueue_ce(d, piece, true, 0); }));
  }
  {
    const int nops = int(S / (size_t(4096) * 8192));  // fits the 8x pitch inside S
    const double b2 = double(nops) * 4096 * 1024 * (G - 1);
    char nm[32];
    std::snprintf(nm, sizeof nm, "2d/%d", nops);
    report(nm, b2, timed([&](int d) { enqueue_2d(d, nops); }));
  }
  // layer-batched 2D copies: per peer, ops of 32 rows of W bytes (one row
  // per layer) into a 2W pitch, the shape of a column-parallel slice of every
  // layer of a replica (7B q: W = 4 MiB, gate/up: 14 MiB)
  for (int wm : {1, 4, 14}) {
    const size_t w = size_t(wm) << 20, rows = 32;
    const int nops = int(S / (2 * w * rows));
    if (nops < 1) continue;
    char nm[32];
    std::snprintf(nm, sizeof nm, "l2d/%dMiBx%d", wm, nops);
    report(nm, double(nops) * w * rows * (G - 1), timed([&](int d) {
             for (int p = 0; p < G; ++p) {
               if (p == d) continue;
               char* to = dst[p] + size_t(d) * S;
               const char* from = src[d] + size_t(p) * S;
               for (int k = 0; k < nops; ++k)
                 CK(cudaMemcpy2DAsync(to + size_t(k) * 2 * w * rows, 2 * w, from + size_t(k) * w * rows, w, w, rows,
                                      cudaMemcpyDefault, st[d][p]));
             }
           }));
  }
  for (int pct : {25, 50, 65, 75}) {
    // CE takes the first pct% (whole pieces per peer), SM the tail
    const size_t ce_bytes = (S / 100 * pct) & ~size_t(4095);
    char nm[32];
    std::snprintf(nm, sizeof nm, "mix/%d", pct);
    report(nm, egress, timed([&](int d) {
             enqueue_ce(d, ce_bytes, true, S - ce_bytes);
             k_a2a<<<ctas, 512, 0, st[d][kMax]>>>(src[d], t, d, G, S, ce_bytes);
           }));
  }
  // H2D from pinned host memory into GPU 0 (and all GPUs at once)
  {
    const size_t hb = size_t(8) << 30;
    void* h = nullptr;
    CK(cudaHostAlloc(&h, hb, cudaHostAllocPortable));
    std::memset(h, 7, hb);
    const int saveG = G;
    for (int all = 0; all <= 1; ++all) {
      for (const char* cfg : {"8192x1", "256x1", "256x2", "256x4", "64x2"}) {
        const size_t piece = size_t(std::atoi(cfg)) << 20;
        const int ns = std::atoi(std::strchr(cfg, 'x') + 1);
        G = all ? saveG : 1;
        const size_t per = std::min(all ? (hb / G) & ~size_t(4095) : hb, saveG * S);
        const double ms = timed([&](int d) {
          char* to = dst[d];
          const char* from = (const char*)h + (all ? size_t(d) * per : 0);
          int i = 0;
          for (size_t off = 0; off < per; off += piece, ++i)
            CK(cudaMemcpyAsync(to + off, from + off, piece < per - off ? piece : per - off,
                               cudaMemcpyHostToDevice, st[d][i % ns]));
        }, 3);
        G = saveG;
        char nm[40];
        std::snprintf(nm, sizeof nm, "h2d%s/%s", all ? "-all" : "", cfg);
        std::printf("%-14s gpus=%d %10.3f ms %8.1f GB/s per GPU, %8.1f GB/s total\n", nm, all ? G : 1, ms,
                    per / (ms * 1e6), (all ? per * G : per) / (ms * 1e6));
        std::fflush(stdout);
      }
    }
    CK(cudaFreeHost(h));
  }
  // verify one a2a delivery (last run direction: h2d overwrote dst[0..]; redo an a2a/ce)
  timed([&](int d) { enqueue_ce(d, S, true, 0); }, 0);
  for (int d = 0; d < G; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceSynchronize());
  }
  int bad = 0;
  for (int d = 0; d < G; ++d)
    for (int p = 0; p < G; ++p) {
      if (p == d) continue;
      unsigned char v = 0;
      CK(cudaMemcpy(&v, dst[d] + size_t(p) * S + S - 1, 1, cudaMemcpyDeviceToHost));
      bad += v != (unsigned char)(p + 1);
    }
  std::printf("check %s\n", bad ? "BAD" : "ok");
  return bad != 0;
}
