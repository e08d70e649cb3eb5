// sm_100a kernels of the reallocation path.
//
//   rr_copy_kernel    K1/K2: descriptor-driven 2D gather -> multi-destination
//                     store. One read of each source chunk, one 16-byte store
//                     per destination (local HBM or a peer-mapped NVLink
//                     address). Replaces the upstream NCCL broadcast plus the
//                     pack/unpack around it.
//   rr_fill_kernel    deterministic bf16 weights from (seed, tensor, index).
//   rr_verify_kernel  regenerate + compare a shard, count mismatches.
//   rr_barrier_kernel cross-GPU flag barrier over peer-mapped memory
//                     (release/acquire at system scope, bounded spin).
#include <cuda_runtime.h>

#include "rr_internal.hpp"

namespace rr {

namespace {

constexpr int kCopyThreads = 256;
constexpr int kCopyUnroll = 8;

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void st_vec(int4* p, const int4& v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Split a flat unit index into (row, col). The float estimate is exact for
// idx < 2^20 (kMaxItemUnits); the two fix-ups make it robust regardless.
__device__ __forceinline__ void split_index(uint32_t idx, uint32_t row_units, float inv,
                                            uint32_t& row, uint32_t& col) {
  row = static_cast<uint32_t>((static_cast<float>(idx) + 0.5f) * inv);
  int32_t c = static_cast<int32_t>(idx - row * row_units);
  if (c < 0) {
    --row;
    c += static_cast<int32_t>(row_units);
  } else if (c >= static_cast<int32_t>(row_units)) {
    ++row;
    c -= static_cast<int32_t>(row_units);
  }
  col = static_cast<uint32_t>(c);
}

// `dsts` points at the shared-memory copy of the item's destination table.
__device__ __forceinline__ void copy_vec_item(const CopyItem& it, const uint64_t* dsts, int ndst,
                                              uint32_t total) {
  const int4* __restrict__ src = reinterpret_cast<const int4*>(it.src);
  const uint32_t step = kCopyThreads * kCopyUnroll;
  for (uint32_t base = 0; base < total; base += step) {
    int4 v[kCopyUnroll];
    uint32_t doff[kCopyUnroll];
#pragma unroll
    for (int u = 0; u < kCopyUnroll; ++u) {
      const uint32_t idx = base + u * kCopyThreads + threadIdx.x;
      doff[u] = 0xffffffffu;
      if (idx < total) {
        uint32_t row, col;
        split_index(idx, it.row_units, it.inv_row, row, col);
        v[u] = ld_stream(src + static_cast<size_t>(row) * it.src_pitch + col);
        doff[u] = row * it.dst_pitch + col;  // < 2^32 units: checked on the host
      }
    }
    for (int j = 0; j < ndst; ++j) {
      int4* dst = reinterpret_cast<int4*>(dsts[j]);
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u)
        if (doff[u] != 0xffffffffu) st_vec(dst + doff[u], v[u]);
    }
  }
}

__device__ __forceinline__ void copy_elem_item(const CopyItem& it, const uint64_t* dsts, int ndst,
                                               uint32_t total) {
  const uint16_t* __restrict__ src = reinterpret_cast<const uint16_t*>(it.src);
  for (uint32_t idx = threadIdx.x; idx < total; idx += kCopyThreads) {
    uint32_t row, col;
    split_index(idx, it.row_units, it.inv_row, row, col);
    const uint16_t v = src[static_cast<size_t>(row) * it.src_pitch + col];
    const size_t off = static_cast<size_t>(row) * it.dst_pitch + col;
    for (int j = 0; j < ndst; ++j) reinterpret_cast<uint16_t*>(dsts[j])[off] = v;
  }
}

__global__ void __launch_bounds__(kCopyThreads) rr_copy_kernel(const CopyItem* __restrict__ items,
                                                               int n_items, int fence_sys) {
  __shared__ CopyItem sh;
  constexpr int kWords = sizeof(CopyItem) / 16;
  for (int i = blockIdx.x; i < n_items; i += gridDim.x) {
    __syncthreads();
    if (threadIdx.x < kWords)
      reinterpret_cast<int4*>(&sh)[threadIdx.x] = reinterpret_cast<const int4*>(items + i)[threadIdx.x];
    __syncthreads();
    CopyItem it;  // scalar fields only; the dst table stays in shared memory
    it.src = sh.src;
    it.row_units = sh.row_units;
    it.nrows = sh.nrows;
    it.src_pitch = sh.src_pitch;
    it.dst_pitch = sh.dst_pitch;
    it.inv_row = sh.inv_row;
    const int ndst = sh.ndst;
    const uint32_t total = it.row_units * it.nrows;
    if (sh.vec)
      copy_vec_item(it, sh.dst, ndst, total);
    else
      copy_elem_item(it, sh.dst, ndst, total);
  }
  // Peer stores must be visible system-wide before a later barrier releases
  // them to the destination GPU.
  if (fence_sys) __threadfence_system();
}

__global__ void rr_fill_kernel(const FillItem* __restrict__ items, int n_items, uint64_t seed) {
  for (int i = blockIdx.x; i < n_items; i += gridDim.x) {
    const FillItem it = items[i];
    uint16_t* base = reinterpret_cast<uint16_t*>(it.base);
    for (uint32_t k = threadIdx.x; k < it.n; k += blockDim.x) {
      const uint32_t e = it.elem0 + k;
      const uint64_t lr = e / it.cols, lc = e % it.cols;
      const uint64_t idx = (it.r0 + lr) * it.full_cols + it.c0 + lc;
      base[e] = weight_value(seed, it.tensor, idx);
    }
  }
}

// counters[0] = mismatches, counters[1] = min buffer element index of a mismatch.
__global__ void rr_verify_kernel(const FillItem* __restrict__ items, int n_items, uint64_t seed,
                                 unsigned long long* counters, uint64_t buf_base) {
  unsigned long long bad = 0, first = ~0ull;
  for (int i = blockIdx.x; i < n_items; i += gridDim.x) {
    const FillItem it = items[i];
    const uint16_t* base = reinterpret_cast<const uint16_t*>(it.base);
    for (uint32_t k = threadIdx.x; k < it.n; k += blockDim.x) {
      const uint32_t e = it.elem0 + k;
      const uint64_t lr = e / it.cols, lc = e % it.cols;
      const uint64_t idx = (it.r0 + lr) * it.full_cols + it.c0 + lc;
      if (base[e] != weight_value(seed, it.tensor, idx)) {
        ++bad;
        const unsigned long long pos = (it.base - buf_base) / 2 + e;
        first = pos < first ? pos : first;
      }
    }
  }
  if (bad) {
    atomicAdd(&counters[0], bad);
    atomicMin(&counters[1], first);
  }
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void rr_barrier_kernel(uint32_t* const* __restrict__ flags, int rank, int world,
                                  uint32_t epoch, int* timed_out) {
  const int p = threadIdx.x;
  if (p < world) {
    __threadfence_system();
    uint32_t* signal = flags[p] + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(signal), "r"(epoch) : "memory");
    const uint32_t* wait = flags[rank] + p;
    const uint64_t t0 = global_ns();
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(wait) : "memory");
      if (static_cast<int32_t>(v - epoch) >= 0) break;
      if (global_ns() - t0 > 20000000000ull) {  // 20 s: report instead of hanging the GPU
        atomicExch(timed_out, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

}  // namespace

int copy_max_ctas(int* ctas_per_sm, int* sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, rr_copy_kernel, kCopyThreads, 0);
}

int launch_copy(const CopyItem* items, int n_items, int ctas, int fence_sys, void* stream) {
  if (n_items <= 0) return cudaSuccess;
  if (ctas > n_items) ctas = n_items;
  rr_copy_kernel<<<ctas, kCopyThreads, 0, static_cast<cudaStream_t>(stream)>>>(items, n_items, fence_sys);
  return cudaGetLastError();
}

int launch_fill(const FillItem* items, int n_items, uint64_t seed, void* stream) {
  if (n_items <= 0) return cudaSuccess;
  const int ctas = n_items < 148 * 16 ? n_items : 148 * 16;
  rr_fill_kernel<<<ctas, 256, 0, static_cast<cudaStream_t>(stream)>>>(items, n_items, seed);
  return cudaGetLastError();
}

int launch_verify(const FillItem* items, int n_items, uint64_t seed, unsigned long long* counters,
                  uint64_t buf_base, void* stream) {
  if (n_items <= 0) return cudaSuccess;
  const int ctas = n_items < 148 * 16 ? n_items : 148 * 16;
  rr_verify_kernel<<<ctas, 256, 0, static_cast<cudaStream_t>(stream)>>>(items, n_items, seed, counters,
                                                                         buf_base);
  return cudaGetLastError();
}

int launch_barrier(uint32_t* const* flags, int rank, int world, uint32_t epoch, int* timed_out,
                   void* stream) {
  rr_barrier_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(flags, rank, world, epoch, timed_out);
  return cudaGetLastError();
}

}  // namespace rr
