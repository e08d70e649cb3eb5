// Copy-engine shapes over NVLink (diagnostics; one process, GPUs 0 and 1,
// both directions at once). Which submissions does a copy engine move at
// full rate when a destination shard's slices are strided per layer?
//   flat             one contiguous copy of the same bytes
//   1d/<n>           n contiguous copies (one per layer)
//   2dL              ONE cudaMemcpy2DAsync: rows = layers (a per-layer slice at a layer stride)
//   2d/<shape>       one cudaMemcpy2DAsync per layer of a row-parallel slice (rows x width, pitches)
//   3d/<shape>       ONE cudaMemcpy3DAsync over all layers of that slice
// Shapes are the plan's real pieces: 70B tp4->tp8 o (8192 x 2 KiB from a
// 4 KiB pitch) and down (8192 x 7 KiB from 14 KiB), 7B tp8->dp8 o (4096 x
// 1 KiB into an 8 KiB pitch) and down (4096 x 3.5 KiB into 28 KiB).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/ce2d_probe tools/ce2d_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) {                                                                \
      std::printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                         \
    }                                                                                       \
  } while (0)

static char* buf_src[2];
static char* buf_dst[2];
static cudaStream_t st[2], st2[2];
static cudaEvent_t ev0[2], ev1[2], evj[2];
static const size_t kBuf = size_t(12) << 30;

// Runs `issue(g, src, dst, stream)` on both GPUs at once (g pushes to 1 - g),
// reps times; prints the slower GPU's GB/s for `bytes` per rep.
static void measure(const char* name, size_t bytes, const std::function<void(int, char*, char*, cudaStream_t)>& issue,
                    int reps = 5) {
  for (int w = 0; w < 2; ++w)
    for (int g = 0; g < 2; ++g) {
      CK(cudaSetDevice(g));
      issue(g, buf_src[g], buf_dst[1 - g], st[g]);
    }
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceSynchronize());
  }
  float worst = 0;
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaEventRecord(ev0[g], st[g]));
    CK(cudaStreamWaitEvent(st2[g], ev0[g], 0));  // the second stream (2-stream modes) starts with the first
  }
  for (int r = 0; r < reps; ++r)
    for (int g = 0; g < 2; ++g) {
      CK(cudaSetDevice(g));
      issue(g, buf_src[g], buf_dst[1 - g], st[g]);
    }
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaEventRecord(evj[g], st2[g]));
    CK(cudaStreamWaitEvent(st[g], evj[g], 0));
    CK(cudaEventRecord(ev1[g], st[g]));
  }
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaEventSynchronize(ev1[g]));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev0[g], ev1[g]));
    if (ms > worst) worst = ms;
  }
  const double per = worst / reps;
  std::printf("%-34s %8.3f ms  %7.1f GB/s per direction  (%.1f MiB per rep)\n", name, per, bytes / (per * 1e-3) / 1e9,
              bytes / 1048576.0);
  std::fflush(stdout);
}

struct Slice {  // a row-parallel slice per layer: rows x width at src/dst pitches, layers at strides
  const char* name;
  size_t rows, width, spitch, dpitch;
};

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    std::printf("needs 2 GPUs\n");
    return 1;
  }
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&buf_src[g], kBuf));
    CK(cudaMalloc(&buf_dst[g], kBuf));
    CK(cudaMemset(buf_src[g], 1, kBuf));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&st2[g], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&evj[g], cudaEventDisableTiming));
    CK(cudaEventCreate(&ev0[g]));
    CK(cudaEventCreate(&ev1[g]));
  }
  int max_pitch = 0;
  CK(cudaDeviceGetAttribute(&max_pitch, cudaDevAttrMaxPitch, 0));
  std::printf("cudaDevAttrMaxPitch %d\n", max_pitch);
  const int L = 40;
  const size_t stride_s = size_t(214) << 20, stride_d = size_t(214) << 20;  // ~70B tp4/tp8 layer strides
  // contiguous per-layer slice (q of 70B tp4 -> tp8: 16 MiB)
  const size_t q = size_t(16) << 20;
  measure("flat 640 MiB", q * L, [&](int, char* s, char* d, cudaStream_t t) {
    CK(cudaMemcpyAsync(d, s, q * L, cudaMemcpyDeviceToDevice, t));
  });
  measure("1d/40 x 16 MiB at layer stride", q * L, [&](int, char* s, char* d, cudaStream_t t) {
    for (int l = 0; l < L; ++l) CK(cudaMemcpyAsync(d + l * stride_d, s + l * stride_s, q, cudaMemcpyDeviceToDevice, t));
  });
  measure("2dL 16 MiB x 40 rows (pitch=stride)", q * L, [&](int, char* s, char* d, cudaStream_t t) {
    CK(cudaMemcpy2DAsync(d, stride_d, s, stride_s, q, L, cudaMemcpyDeviceToDevice, t));
  });
  measure("1d/40 x 16 MiB, 2 streams alternating", q * L, [&](int g, char* s, char* d, cudaStream_t t) {
    for (int l = 0; l < L; ++l)
      CK(cudaMemcpyAsync(d + l * stride_d, s + l * stride_s, q, cudaMemcpyDeviceToDevice, (l & 1) ? st2[g] : t));
  });
  // back-to-back 2D copies like the 34B / 70B transport's (one tensor kind of
  // a stage: 16 MiB rows x 12 layers), 10 in a row, on one and on two streams
  measure("2dL 16 MiB x 12 rows, 10 copies", q * 120, [&](int, char* s, char* d, cudaStream_t t) {
    for (int k = 0; k < 10; ++k)
      CK(cudaMemcpy2DAsync(d + k * q, stride_d, s + k * q, stride_s, q, 12, cudaMemcpyDeviceToDevice, t));
  });
  measure("2dL 16 MiB x 12 rows, 10 copies, 2 streams", q * 120, [&](int g, char* s, char* d, cudaStream_t t) {
    for (int k = 0; k < 10; ++k)
      CK(cudaMemcpy2DAsync(d + k * q, stride_d, s + k * q, stride_s, q, 12, cudaMemcpyDeviceToDevice,
                           (k & 1) ? st2[g] : t));
  });
  measure("2dL 4 MiB x 12 rows, 40 copies", q * 120, [&](int, char* s, char* d, cudaStream_t t) {
    const size_t w = q / 4;
    for (int k = 0; k < 40; ++k)
      CK(cudaMemcpy2DAsync(d + k * w, stride_d, s + k * w, stride_s, w, 12, cudaMemcpyDeviceToDevice, t));
  });
  measure("2dL 4 MiB x 12 rows, 40 copies, 2 streams", q * 120, [&](int g, char* s, char* d, cudaStream_t t) {
    const size_t w = q / 4;
    for (int k = 0; k < 40; ++k)
      CK(cudaMemcpy2DAsync(d + k * w, stride_d, s + k * w, stride_s, w, 12, cudaMemcpyDeviceToDevice,
                           (k & 1) ? st2[g] : t));
  });
  const size_t small = size_t(1) << 20;  // 7B k slice (1 MiB) x 32 layers
  measure("1d/32 x 1 MiB at layer stride", small * 32, [&](int, char* s, char* d, cudaStream_t t) {
    for (int l = 0; l < 32; ++l)
      CK(cudaMemcpyAsync(d + l * stride_d, s + l * stride_s, small, cudaMemcpyDeviceToDevice, t));
  });
  measure("2dL 1 MiB x 32 rows", small * 32, [&](int, char* s, char* d, cudaStream_t t) {
    CK(cudaMemcpy2DAsync(d, stride_d, s, stride_s, small, 32, cudaMemcpyDeviceToDevice, t));
  });
  const Slice shapes[] = {{"70B o   8192 x 2 KiB (4K->2K)", 8192, 2048, 4096, 2048},
                          {"70B down 8192 x 7 KiB (14K->7K)", 8192, 7168, 14336, 7168},
                          {"7B o    4096 x 1 KiB (1K->8K)", 4096, 1024, 1024, 8192},
                          {"7B down 4096 x 3.5 KiB (3.5K->28K)", 4096, 3584, 3584, 28672}};
  for (const Slice& sh : shapes) {
    const size_t bytes = sh.rows * sh.width * L;
    // layer strides that are whole multiples of the pitches (3D needs slice pitch = pitch x height)
    const size_t ys = (stride_s + sh.spitch - 1) / sh.spitch, yd = (stride_d + sh.dpitch - 1) / sh.dpitch;
    std::string n2 = std::string("2d/40 ") + sh.name, n3 = std::string("3d ") + sh.name;
    measure(n2.c_str(), bytes, [&](int, char* s, char* d, cudaStream_t t) {
      for (int l = 0; l < L; ++l)
        CK(cudaMemcpy2DAsync(d + l * yd * sh.dpitch, sh.dpitch, s + l * ys * sh.spitch, sh.spitch, sh.width, sh.rows,
                             cudaMemcpyDeviceToDevice, t));
    });
    measure(n3.c_str(), bytes, [&](int, char* s, char* d, cudaStream_t t) {
      cudaMemcpy3DParms p = {};
      p.srcPtr = make_cudaPitchedPtr(s, sh.spitch, sh.width, ys);
      p.dstPtr = make_cudaPitchedPtr(d, sh.dpitch, sh.width, yd);
      p.extent = make_cudaExtent(sh.width, sh.rows, L);
      p.kind = cudaMemcpyDeviceToDevice;
      CK(cudaMemcpy3DAsync(&p, t));
    });
  }
  return 0;
}
