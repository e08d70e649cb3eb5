// Strided multi-destination store probe (diagnostics; one GPU).
// The row-parallel tensors (o, down) of a tp -> dp reallocation land in each
// destination as R rows of W bytes at a pitch of P bytes. How fast can one
// source read feed 8 such destinations? (HBM bytes = read + 8 x write.)
//   bulk_rows   TMA ring, one cp.async.bulk shared->global per row per dst
//               (what rr_bulk_kernel does for strided pieces)
//   bulk_flat   the same bytes stored contiguously (no pitch): the ceiling
//   tensor      TMA ring, one cp.async.bulk.tensor.2d store per piece per dst
//               (a CUtensorMap per destination describes rows x pitch)
//   ldst        registers: 16 B ld.global.nc / st.global per thread
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/strided_probe \
//          tools/strided_probe.cu -L/usr/local/cuda/lib64/stubs -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) {                                                                   \
      std::printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));   \
      std::exit(1);                                                                            \
    }                                                                                          \
  } while (0)

constexpr int kDst = 8;
constexpr int kStage = 16384, kS = 4;

struct Dsts {
  uint64_t p[kDst];
};
struct Maps {
  CUtensorMap m[kDst];
};

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// mode 0: per-row stores with pitch; 1: flat stores; 2: tensor stores
template <int MODE>
__global__ void __launch_bounds__(32) k_ring(const char* __restrict__ src, Dsts d, const __grid_constant__ Maps maps,
                                             size_t bytes, uint32_t row, uint32_t pitch) {
  extern __shared__ __align__(1024) char ring[];
  __shared__ __align__(8) uint64_t bar[kS];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t pieces = bytes / kStage;
  const uint32_t rows_per = kStage / row;
  uint32_t ph[kS] = {0, 0, 0, 0};
  size_t ld = blockIdx.x;
  int issued = 0;
  auto issue = [&](int s) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(kStage));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa(ring + s * kStage)),
                 "l"(src + ld * kStage), "r"(kStage), "r"(sa(&bar[s]))
                 : "memory");
  };
  size_t piece_of[kS];
  for (int s = 0; s < kS && ld < pieces; ++s, ld += gridDim.x, ++issued) {
    piece_of[s] = ld;
    issue(s);
  }
  for (int done = 0; done < issued; ++done) {
    const int s = done % kS;
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(
                     sa(&bar[s])),
                 "r"(ph[s]));
    ph[s] ^= 1;
    const size_t pc = piece_of[s];
    const uint32_t r0 = (uint32_t)(pc * rows_per);
    for (int j = 0; j < kDst; ++j) {
      if (MODE == 1) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d.p[j] + pc * kStage),
                     "r"(sa(ring + s * kStage)), "r"(kStage)
                     : "memory");
      } else if (MODE == 0) {
        for (uint32_t r = 0; r < rows_per; ++r)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                           d.p[j] + (uint64_t)(r0 + r) * pitch),
                       "r"(sa(ring + s * kStage + r * row)), "r"(row)
                       : "memory");
      } else {
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&maps.m[j]),
                     "r"(0), "r"(r0), "r"(sa(ring + s * kStage))
                     : "memory");
      }
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (done >= 1) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      if (ld < pieces) {
        const int f = (done - 1) % kS;
        piece_of[f] = ld;
        issue(f);
        ld += gridDim.x;
        ++issued;
      }
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(256) k_ldst(const int4* __restrict__ src, Dsts d, size_t n16, uint32_t row16,
                                              uint32_t pitch16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    const int4 v = __ldg(src + i);
    const size_t r = i / row16, c = i % row16;
#pragma unroll
    for (int j = 0; j < kDst; ++j) reinterpret_cast<int4*>(d.p[j])[r * pitch16 + c] = v;
  }
}

int main(int argc, char** argv) {
  const uint32_t row = argc > 1 ? (uint32_t)std::atoi(argv[1]) : 1024;  // bytes per row
  const uint32_t pitch = argc > 2 ? (uint32_t)std::atoi(argv[2]) : 8192;
  const size_t bytes = size_t(1) << 30;  // source bytes
  const size_t rows = bytes / row;
  char* src;
  CK(cudaMalloc(&src, bytes));
  CK(cudaMemset(src, 7, bytes));
  Dsts d;
  for (int j = 0; j < kDst; ++j) {
    void* p;
    CK(cudaMalloc(&p, rows * pitch));
    d.p[j] = (uint64_t)p;
  }
  Maps maps;
  std::memset(&maps, 0, sizeof(maps));
  for (int j = 0; j < kDst; ++j) {
    cuuint64_t dims[2] = {row / 8, rows};  // 8-byte elements
    cuuint64_t strides[1] = {pitch};
    cuuint32_t box[2] = {row / 8, kStage / row};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&maps.m[j], CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, (void*)d.p[j], dims, strides,
                                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      std::printf("tensor map encode failed %d (row %u)\n", (int)r, row);
      return 1;
    }
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(k_ring<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kS * kStage));
  CK(cudaFuncSetAttribute(k_ring<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kS * kStage));
  CK(cudaFuncSetAttribute(k_ring<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kS * kStage));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const double traffic = (double)bytes * (1 + kDst);
  for (int mode = 0; mode < 4; ++mode) {
    for (int mult : {3, 4, 6}) {
      if (mode == 3 && mult != 3) continue;
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(a));
        if (mode == 0) k_ring<0><<<sms * mult, 32, kS * kStage>>>(src, d, maps, bytes, row, pitch);
        if (mode == 1) k_ring<1><<<sms * mult, 32, kS * kStage>>>(src, d, maps, bytes, row, pitch);
        if (mode == 2) k_ring<2><<<sms * mult, 32, kS * kStage>>>(src, d, maps, bytes, row, pitch);
        if (mode == 3) k_ldst<<<sms * 8, 256>>>((const int4*)src, d, bytes / 16, row / 16, pitch / 16);
        CK(cudaGetLastError());
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (rep > 0 && ms < best) best = ms;
      }
      const char* nm[] = {"bulk_rows", "bulk_flat", "tensor", "ldst"};
      std::printf("row=%u pitch=%u %-9s ctas/SM=%d %8.1f GB/s (read + 8 x write)\n", row, pitch, nm[mode],
                  mode == 3 ? 8 : mult, traffic / (best * 1e6));
    }
  }
  // check: tensor mode wrote row r of dst 7 correctly
  CK(cudaMemset((void*)d.p[7], 0, rows * pitch));
  k_ring<2><<<sms * 3, 32, kS * kStage>>>(src, d, maps, bytes, row, pitch);
  CK(cudaDeviceSynchronize());
  unsigned char h[2];
  CK(cudaMemcpy(&h[0], (char*)d.p[7] + (rows - 1) * pitch + row - 1, 1, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&h[1], (char*)d.p[7] + (rows - 1) * pitch + row, 1, cudaMemcpyDeviceToHost));
  std::printf("check %s\n", (h[0] == 7 && h[1] == 0) ? "ok" : "BAD");
  return 0;
}
