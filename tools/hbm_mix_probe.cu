// HBM traffic-mix probe (diagnostics; one GPU).
// What is the ceiling for the 1:8 read:write mix of the 7B train->gen
// reallocation (one source shard read once, stored into 8 replicas), and
// which store mechanism gets closest to it?
//   w/*    pure writes over 64 GiB: TMA bulk stores of a constant smem tile,
//          st.global.v4 / v8 from registers, cudaMemsetAsync
//   r/*    pure reads over 64 GiB: TMA bulk loads into a ring, ld.global.nc v4
//   cp/*   1:1 copy 32 GiB -> 32 GiB
//   bc/*   1:8 broadcast 8 GiB -> 8 x 8 GiB (src read once)
//          tma<S,K>    ring of S stages of K bytes; each stage stored to all 8
//                      destinations before the next (the product's order)
//          tmadst<S,K> S stages loaded, then stored destination-major (all
//                      stages to dst 0, then dst 1, ...): longer write runs
//          reg         registers: ld.v4 x8 unrolled, 8 stores each
// GB/s = (bytes read + bytes written) / time; best of 5 after a warm-up.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/hbm_mix_probe tools/hbm_mix_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) {                                                                \
      std::printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                         \
    }                                                                                       \
  } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sa(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void bload(void* s, const void* g, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(s)),
               "l"(g), "r"(n), "r"(sa(b))
               : "memory");
}
__device__ __forceinline__ void bstore(void* g, const void* s, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(sa(s)), "r"(n) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// ---- pure writes ----
template <int K>
__global__ void __launch_bounds__(32) w_tma(char* dst, size_t chunks) {
  extern __shared__ __align__(128) uint8_t tile[];
  for (int i = threadIdx.x; i < K / 16; i += 32) reinterpret_cast<int4*>(tile)[i] = make_int4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (threadIdx.x) return;
  int n = 0;
  for (size_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    bstore(dst + c * K, tile, K);
    commit();
    if (++n >= 8) wait_read<7>();
  }
  wait_all();
}

__global__ void w_v4(int4* dst, size_t n) {
  const int4 z = make_int4(1, 2, 3, 4);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) dst[i] = z;
}

__global__ void w_v8(int4* dst, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; 2 * i < n16; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(dst + 2 * i), "r"(7) : "memory");
}

// ---- pure reads ----
template <int S, int K>
__global__ void __launch_bounds__(32) r_tma(const char* src, size_t chunks) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[S];
  if (threadIdx.x) return;
  for (int s = 0; s < S; ++s) mbar_init(&full[s]);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  size_t issued = 0, done = 0;
  size_t c = blockIdx.x;
  for (;;) {
    while (issued - done < S && c < chunks) {
      const int s = issued % S;
      mbar_expect(&full[s], K);
      bload(ring + s * K, src + c * K, K, &full[s]);
      ++issued;
      c += gridDim.x;
    }
    if (done == issued) break;
    mbar_wait(&full[done % S], (done / S) & 1);
    ++done;
  }
}

__global__ void r_v4(const int4* src, size_t n, int* sink) {
  int acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(src + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x7fffffff) *sink = acc;
}

// ---- copy / broadcast through a TMA ring ----
struct Dsts {
  char* d[8];
};

// ND destinations; DSTMAJOR: drain all S stages per destination in turn.
template <int S, int K, int ND, bool DSTMAJOR>
__global__ void __launch_bounds__(32) bc_tma(const char* src, Dsts dsts, size_t chunks) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[S];
  if (threadIdx.x) return;
  for (int s = 0; s < S; ++s) mbar_init(&full[s]);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (!DSTMAJOR) {
    size_t issued = 0, done = 0, c = blockIdx.x;
    size_t cidx[S];
    for (;;) {
      while ((issued < S || issued - done < S - 1) && c < chunks) {
        if (issued >= S) wait_read<1>();
        const int s = issued % S;
        cidx[s] = c;
        mbar_expect(&full[s], K);
        bload(ring + s * K, src + c * K, K, &full[s]);
        ++issued;
        c += gridDim.x;
      }
      if (done == issued) break;
      const int s = done % S;
      mbar_wait(&full[s], (done / S) & 1);
      for (int j = 0; j < ND; ++j) bstore(dsts.d[j] + cidx[s] * K, ring + s * K, K);
      commit();
      ++done;
    }
  } else {
    // batches of S consecutive-in-this-CTA chunks: load all, then per destination store all
    uint32_t phase = 0;
    for (size_t c0 = size_t(blockIdx.x) * S; c0 < chunks; c0 += size_t(gridDim.x) * S) {
      const int n = (int)(chunks - c0 < S ? chunks - c0 : S);
      wait_read<0>();
      for (int s = 0; s < n; ++s) {
        mbar_expect(&full[s], K);
        bload(ring + s * K, src + (c0 + s) * K, K, &full[s]);
      }
      for (int s = 0; s < n; ++s) mbar_wait(&full[s], phase);
      for (int j = 0; j < ND; ++j) {
        bstore(dsts.d[j] + c0 * K, ring, n * K);
        commit();
      }
      phase ^= 1;
    }
  }
  wait_all();
}

__global__ void bc_reg(const int4* src, Dsts dsts, size_t n) {
  constexpr int U = 4;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t b = blockIdx.x * (size_t)blockDim.x + threadIdx.x; b < n; b += stride * U) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (b + u * stride < n)
        asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(src + b + u * stride));
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (b + u * stride < n) reinterpret_cast<int4*>(dsts.d[j])[b + u * stride] = v[u];
  }
}

// 32-byte loads and stores; U independent loads in flight per thread.
template <int U>
__global__ void bc_reg8(const int4* src, Dsts dsts, size_t n32) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t b = blockIdx.x * (size_t)blockDim.x + threadIdx.x; b < n32; b += stride * U) {
    uint32_t r[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (b + u * stride < n32)
        asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[u][0]), "=r"(r[u][1]), "=r"(r[u][2]), "=r"(r[u][3]), "=r"(r[u][4]), "=r"(r[u][5]),
                       "=r"(r[u][6]), "=r"(r[u][7])
                     : "l"(src + 2 * (b + u * stride)));
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (b + u * stride < n32)
          asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(
                           reinterpret_cast<int4*>(dsts.d[j]) + 2 * (b + u * stride)),
                       "r"(r[u][0]), "r"(r[u][1]), "r"(r[u][2]), "r"(r[u][3]), "r"(r[u][4]), "r"(r[u][5]),
                       "r"(r[u][6]), "r"(r[u][7])
                       : "memory");
  }
}

// Hybrid: thread 0 streams K-byte chunks into a 2-stage smem ring with TMA
// loads; all warps store each stage to the 8 destinations with st.global.v8.
template <int K>
__global__ void __launch_bounds__(512) bc_hyb(const char* src, Dsts dsts, size_t chunks) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[2];
  if (threadIdx.x == 0) {
    mbar_init(&full[0]);
    mbar_init(&full[1]);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  size_t c = blockIdx.x;
  if (threadIdx.x == 0 && c < chunks) {
    mbar_expect(&full[0], K);
    bload(ring, src + c * K, K, &full[0]);
  }
  for (int it = 0; c < chunks; ++it, c += gridDim.x) {
    const int s = it & 1;
    const size_t cn = c + gridDim.x;
    if (threadIdx.x == 0 && cn < chunks) {  // prefetch the next chunk into the other stage
      mbar_expect(&full[s ^ 1], K);
      bload(ring + (s ^ 1) * K, src + cn * K, K, &full[s ^ 1]);
    }
    mbar_wait(&full[s], (it >> 1) & 1);
    const uint4* t = reinterpret_cast<const uint4*>(ring + s * K);
    for (int i = threadIdx.x; i < K / 32; i += blockDim.x) {
      const uint4 a = t[2 * i], b = t[2 * i + 1];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dsts.d[j] + c * K + 32 * i), "r"(a.x),
                     "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                     : "memory");
    }
    __syncthreads();  // stage s is free before it is refilled two chunks later
  }
}

// Run-partitioned variants: a CTA claims runs of R contiguous bytes from an
// atomic counter (as the product's items) and streams each run in K-byte
// chunks. ctr[0] must be zero at launch; the last CTA out resets it.
template <int S, int K, int ND>
__global__ void __launch_bounds__(32) bc_run(const char* src, Dsts dsts, size_t bytes, size_t run,
                                             unsigned int* ctr) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[S];
  if (threadIdx.x) return;
  for (int s = 0; s < S; ++s) mbar_init(&full[s]);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const size_t nruns = (bytes + run - 1) / run;
  size_t r = atomicAdd(ctr, 1u), off = 0;
  size_t issued = 0, done = 0;
  size_t cpos[S];
  for (;;) {
    while ((issued < S || issued - done < S - 1) && r < nruns) {
      if (issued >= S) wait_read<1>();
      const int s = issued % S;
      cpos[s] = r * run + off;
      mbar_expect(&full[s], K);
      bload(ring + s * K, src + cpos[s], K, &full[s]);
      ++issued;
      off += K;
      if (off >= run || r * run + off >= bytes) {
        off = 0;
        r = atomicAdd(ctr, 1u);
      }
    }
    if (done == issued) break;
    const int s = done % S;
    mbar_wait(&full[s], (done / S) & 1);
    for (int j = 0; j < ND; ++j) bstore(dsts.d[j] + cpos[s], ring + s * K, K);
    commit();
    ++done;
  }
  wait_all();
  __threadfence();
  if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
    atomicExch(ctr, 0u);
    atomicExch(ctr + 1, 0u);
  }
}

__global__ void w_v8_run(char* dst, size_t bytes, size_t run, unsigned int* ctr) {
  __shared__ size_t r;
  const size_t nruns = (bytes + run - 1) / run;
  for (;;) {
    if (threadIdx.x == 0) r = atomicAdd(ctr, 1u);
    __syncthreads();
    const size_t my = r;
    __syncthreads();
    if (my >= nruns) break;
    char* base = dst + my * run;
    for (size_t i = threadIdx.x * 32; i < run; i += blockDim.x * 32)
      asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(base + i), "r"(7) : "memory");
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
      atomicExch(ctr, 0u);
      atomicExch(ctr + 1, 0u);
    }
  }
}

// Register broadcast over claimed runs: 32-byte loads, 8 x 32-byte stores.
template <int U>
__global__ void __launch_bounds__(512) bc_reg8_run(const char* src, Dsts dsts, size_t bytes, size_t run,
                                                  unsigned int* ctr) {
  __shared__ size_t r;
  const size_t nruns = (bytes + run - 1) / run;
  for (;;) {
    if (threadIdx.x == 0) r = atomicAdd(ctr, 1u);
    __syncthreads();
    const size_t my = r;
    __syncthreads();
    if (my >= nruns) break;
    const size_t base = my * run;
    for (size_t i0 = threadIdx.x * 32; i0 < run; i0 += size_t(blockDim.x) * 32 * U) {
      uint32_t v[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t i = i0 + size_t(u) * blockDim.x * 32;
        if (i < run)
          asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(v[u][0]), "=r"(v[u][1]), "=r"(v[u][2]), "=r"(v[u][3]), "=r"(v[u][4]), "=r"(v[u][5]),
                         "=r"(v[u][6]), "=r"(v[u][7])
                       : "l"(src + base + i));
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const size_t i = i0 + size_t(u) * blockDim.x * 32;
          if (i < run)
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dsts.d[j] + base + i), "r"(v[u][0]),
                         "r"(v[u][1]), "r"(v[u][2]), "r"(v[u][3]), "r"(v[u][4]), "r"(v[u][5]), "r"(v[u][6]),
                         "r"(v[u][7])
                         : "memory");
        }
    }
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
      atomicExch(ctr, 0u);
      atomicExch(ctr + 1, 0u);
    }
  }
}

template <int K>
__global__ void __launch_bounds__(32) w_tma_run(char* dst, size_t bytes, size_t run, unsigned int* ctr) {
  extern __shared__ __align__(128) uint8_t tile[];
  for (int i = threadIdx.x; i < K / 16; i += 32) reinterpret_cast<int4*>(tile)[i] = make_int4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (threadIdx.x) return;
  const size_t nruns = (bytes + run - 1) / run;
  int n = 0;
  for (size_t r = atomicAdd(ctr, 1u); r < nruns; r = atomicAdd(ctr, 1u))
    for (size_t off = 0; off < run; off += K) {
      bstore(dst + r * run + off, tile, K);
      commit();
      if (++n >= 8) wait_read<7>();
    }
  wait_all();
  __threadfence();
  if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
    atomicExch(ctr, 0u);
    atomicExch(ctr + 1, 0u);
  }
}


// Phase-separated broadcast: every CTA loads its slice of a round into
// shared memory, a grid-wide barrier, then stores it to the 8 destinations
// and waits for the stores to complete, another barrier. DRAM then sees
// long pure-read and pure-write periods instead of a fine-grained mix.
__device__ __forceinline__ void grid_sync(unsigned int* bar, unsigned int& gen) {
  __syncwarp();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int target = (gen + 1) * gridDim.x;
    atomicAdd(bar, 1u);
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {  // bounded: a wrong occupancy must not hang the GPU
      unsigned int v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (v >= target) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 2000000000ull) break;
    }
  }
  ++gen;
  __syncwarp();
}

__global__ void __launch_bounds__(32) bc_phased(const char* src, Dsts dsts, size_t bytes, unsigned int* bar,
                                                uint32_t per_cta, int barriers) {
  extern __shared__ __align__(128) uint8_t buf[];
  __shared__ __align__(8) uint64_t full;
  unsigned int gen = 0;
  if (threadIdx.x == 0) {
    mbar_init(&full);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  const size_t round_bytes = size_t(per_cta) * gridDim.x;
  uint32_t phase = 0;
  for (size_t base = 0; base < bytes; base += round_bytes) {
    const size_t off = base + size_t(blockIdx.x) * per_cta;
    const uint32_t n = off < bytes ? (uint32_t)min(size_t(per_cta), bytes - off) : 0;
    if (threadIdx.x == 0 && n) {
      mbar_expect(&full, n);
      for (uint32_t k = 0; k < n; k += 32768) bload(buf + k, src + off + k, min(32768u, n - k), &full);
      mbar_wait(&full, phase);
    }
    phase ^= n ? 1 : 0;
    if (barriers) grid_sync(bar, gen);
    if (threadIdx.x == 0 && n) {
      for (int j = 0; j < 8; ++j) bstore(dsts.d[j] + off, buf, n);
      commit();
      wait_all();
    }
    if (barriers) grid_sync(bar, gen);
  }
}

static cudaEvent_t t0, t1;

template <class F>
static double best_ms(F&& f) {
  double best = 1e30;
  for (int r = 0; r < 6; ++r) {
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(t0));
    f();
    CK(cudaGetLastError());
    CK(cudaEventRecord(t1));
    CK(cudaEventSynchronize(t1));
    float m = 0;
    CK(cudaEventElapsedTime(&m, t0, t1));
    if (r && m < best) best = m;
  }
  return best;
}

static void rep(const char* name, int ctas, double bytes, double ms) {
  std::printf("%-22s ctas=%-5d %8.3f ms %8.1f GB/s\n", name, ctas, ms, bytes / (ms * 1e6));
  std::fflush(stdout);
}

template <int S, int K, int ND, bool DM>
static void run_bc(const char* name, const char* src, Dsts d, size_t bytes, int sms) {
  const int smem = S * K;
  CK(cudaFuncSetAttribute(bc_tma<S, K, ND, DM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bc_tma<S, K, ND, DM>, 32, smem));
  for (int m = 1; m <= per && m <= 4; ++m) {
    const int ctas = sms * m;
    const double ms = best_ms([&] { bc_tma<S, K, ND, DM><<<ctas, 32, smem>>>(src, d, bytes / K); });
    rep(name, ctas, double(bytes) * (1 + ND), ms);
  }
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  const size_t G = size_t(1) << 30;
  const size_t big = 64 * G, sb = 8 * G;
  char *a = nullptr, *s = nullptr;
  int* sink = nullptr;
  CK(cudaMalloc(&a, big));
  CK(cudaMalloc(&s, sb));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(s, 3, sb));
  CK(cudaMemset(a, 1, big));
  rep("w/memset-nz", 0, big, best_ms([&] { CK(cudaMemsetAsync(a, 0x5a, big)); }));

  rep("w/memset", 0, big, best_ms([&] { CK(cudaMemsetAsync(a, 0, big)); }));
  for (int m : {1, 8, 16, 32}) {
    rep("w/v4", sms * m, big, best_ms([&] { w_v4<<<sms * m, 512>>>((int4*)a, big / 16); }));
    rep("w/v8", sms * m, big, best_ms([&] { w_v8<<<sms * m, 512>>>((int4*)a, big / 16); }));
  }
  CK(cudaFuncSetAttribute(w_tma<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  CK(cudaFuncSetAttribute(w_tma<65536>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  for (int m : {1, 2, 4}) {
    rep("w/tma16k", sms * m, big, best_ms([&] { w_tma<16384><<<sms * m, 32, 16384>>>(a, big / 16384); }));
    rep("w/tma64k", sms * m, big, best_ms([&] { w_tma<65536><<<sms * m, 32, 65536>>>(a, big / 65536); }));
  }
  for (int m : {1, 2, 4, 8})
    rep("r/v4", sms * m, big, best_ms([&] { r_v4<<<sms * m, 512>>>((const int4*)a, big / 16, sink); }));
  CK(cudaFuncSetAttribute(r_tma<4, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384));
  CK(cudaFuncSetAttribute(r_tma<4, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768));
  for (int m : {1, 2, 3}) {
    rep("r/tma4x16k", sms * m, big, best_ms([&] { r_tma<4, 16384><<<sms * m, 32, 4 * 16384>>>(a, big / 16384); }));
    rep("r/tma4x32k", sms * m, big, best_ms([&] { r_tma<4, 32768><<<sms * m, 32, 4 * 32768>>>(a, big / 32768); }));
  }
  // 1:1 copy, 32 GiB -> 32 GiB
  {
    Dsts d{};
    d.d[0] = a + 32 * G;
    run_bc<4, 16384, 1, false>("cp/tma4x16k", a, d, 32 * G, sms);
    run_bc<4, 32768, 1, false>("cp/tma4x32k", a, d, 32 * G, sms);
    const double ms = best_ms([&] { CK(cudaMemcpyAsync(a + 32 * G, a, 32 * G, cudaMemcpyDeviceToDevice)); });
    rep("cp/cudaMemcpy", 0, 64.0 * G, ms);
  }
  // 1:8 broadcast, 8 GiB -> 8 x 8 GiB; destinations first at a power-of-two
  // stride (8 GiB apart), then at the product's kind of stride (replicas
  // 16.06 GB apart: here 3.5 GiB + 12.25 MiB + 256 B) to see address aliasing
  Dsts d{};
  for (int j = 0; j < 8; ++j) d.d[j] = a + j * sb;
  run_bc<4, 16384, 8, false>("bc/tma4x16k/pow2", s, d, sb, sms);
  const size_t sbo = 3 * G + G / 2;  // 3.5 GiB source so that everything fits in 64 GiB
  const size_t odd = sbo + (size_t(49) << 18) + 256;
  CK(cudaFree(s));
  s = a + 8 * odd;  // the source sits after the destinations inside `a`
  for (int j = 0; j < 8; ++j) d.d[j] = a + j * odd;
  CK(cudaMemset(s, 3, sbo));
  run_bc<4, 16384, 8, false>("bc/tma4x16k", s, d, sbo, sms);
  run_bc<3, 16384, 8, false>("bc/tma3x16k", s, d, sbo, sms);
  run_bc<2, 65536, 8, false>("bc/tma2x64k", s, d, sbo, sms);
  run_bc<4, 16384, 8, true>("bc/tmadst4x16k", s, d, sbo, sms);
  run_bc<4, 32768, 8, true>("bc/tmadst4x32k", s, d, sbo, sms);
  for (int m : {1, 4, 8})
    rep("bc/reg", sms * m, 9.0 * sbo, best_ms([&] { bc_reg<<<sms * m, 256>>>((const int4*)s, d, sbo / 16); }));
  for (int m : {2, 4, 8, 16}) {
    rep("bc/reg8u1", sms * m, 9.0 * sbo, best_ms([&] { bc_reg8<1><<<sms * m, 256>>>((const int4*)s, d, sbo / 32); }));
    rep("bc/reg8u2", sms * m, 9.0 * sbo, best_ms([&] { bc_reg8<2><<<sms * m, 256>>>((const int4*)s, d, sbo / 32); }));
  }
  CK(cudaFuncSetAttribute(bc_hyb<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 16384));
  CK(cudaFuncSetAttribute(bc_hyb<32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 32768));
  for (int m : {1, 2, 3, 4}) {
    rep("bc/hyb16k", sms * m, 9.0 * sbo, best_ms([&] { bc_hyb<16384><<<sms * m, 512, 2 * 16384>>>(s, d, sbo / 16384); }));
    rep("bc/hyb32k", sms * m, 9.0 * sbo, best_ms([&] { bc_hyb<32768><<<sms * m, 512, 2 * 32768>>>(s, d, sbo / 32768); }));
  }
  unsigned int* ctr = nullptr;
  CK(cudaMalloc(&ctr, 8));
  CK(cudaMemset(ctr, 0, 8));
  CK(cudaFuncSetAttribute(bc_run<4, 16384, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384));
  CK(cudaFuncSetAttribute(bc_run<4, 32768, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768));
  CK(cudaFuncSetAttribute(w_tma_run<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  for (size_t run : {size_t(16) << 10, size_t(32) << 10, size_t(64) << 10, size_t(256) << 10}) {
    char nm[40];
    for (int m : {1, 2}) {
      std::snprintf(nm, sizeof nm, "bc/run%zuk/4x16k", run >> 10);
      rep(nm, sms * m, 9.0 * sbo,
          best_ms([&] { bc_run<4, 16384, 8><<<sms * m, 32, 4 * 16384>>>(s, d, sbo, run, ctr); }));
    }
    if (run >= 32768) {
      std::snprintf(nm, sizeof nm, "bc/run%zuk/4x32k", run >> 10);
      rep(nm, sms, 9.0 * sbo, best_ms([&] { bc_run<4, 32768, 8><<<sms, 32, 4 * 32768>>>(s, d, sbo, run, ctr); }));
    }
    for (int m : {2, 4, 8}) {
      std::snprintf(nm, sizeof nm, "bc/reg8u1run%zuk", run >> 10);
      rep(nm, sms * m, 9.0 * sbo, best_ms([&] { bc_reg8_run<1><<<sms * m, 512>>>(s, d, sbo, run, ctr); }));
      std::snprintf(nm, sizeof nm, "bc/reg8u2run%zuk", run >> 10);
      rep(nm, sms * m, 9.0 * sbo, best_ms([&] { bc_reg8_run<2><<<sms * m, 512>>>(s, d, sbo, run, ctr); }));
    }
    for (int m : {1, 2, 4}) {
      std::snprintf(nm, sizeof nm, "w/tmarun%zuk", run >> 10);
      rep(nm, sms * m, double(32 * G), best_ms([&] { w_tma_run<16384><<<sms * m, 32, 16384>>>(a + 32 * G, 32 * G, run, ctr); }));
    }
    std::snprintf(nm, sizeof nm, "w/v8run%zuk", run >> 10);
    rep(nm, sms * 4, double(32 * G), best_ms([&] { w_v8_run<<<sms * 4, 512>>>(a + 32 * G, 32 * G, run, ctr); }));
  }
  unsigned int* bar = nullptr;
  CK(cudaMalloc(&bar, 4));
  for (uint32_t per : {65536u, 98304u, 196608u}) {
    CK(cudaFuncSetAttribute(bc_phased, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bc_phased, 32, per));
    for (int barriers : {1, 0}) {
      const int ctas = sms * occ;  // all resident: the grid barrier needs it
      char nm[40];
      std::snprintf(nm, sizeof nm, "bc/phased%uk%s", per >> 10, barriers ? "" : "-nobar");
      rep(nm, ctas, 9.0 * sbo, best_ms([&] {
            CK(cudaMemsetAsync(bar, 0, 4));
            bc_phased<<<ctas, 32, per>>>(s, d, sbo, bar, per, barriers);
          }));
    }
  }
  // check the last broadcast: every destination equals the source pattern (0x03)
  unsigned char h[2] = {0, 0};
  CK(cudaMemcpy(&h[0], d.d[7] + sbo - 1, 1, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&h[1], d.d[0], 1, cudaMemcpyDeviceToHost));
  std::printf("check %s\n", (h[0] == 3 && h[1] == 3) ? "ok" : "BAD");
  return 0;
}
