// 1:8 broadcast vs L2 (diagnostics; one GPU). Where does the gap between the
// 1:8 broadcast (6.59 TB/s, profiles/r01_hbm_mix_probe.txt) and pure writes
// (7.4 TB/s) come from, and does staging the source through L2 close it?
//   base        the product's scheme: CTAs claim 16 KiB runs in address order,
//               TMA ring 4 x 16 KiB, each stage stored to 8 destinations
//   srcL2/W     the same, but the source offset wraps inside a W-byte window,
//               so loads hit L2: the DRAM sees (almost) only the 8 write streams
//   pf/A        base + cp.async.bulk.prefetch.L2 of the source A bytes ahead of
//               the run being loaded (reads become early, non-blocking L2 fills)
//   stEF        base with L2::evict_first on the stores
//   dmaj/W      destination-major: the source is cut into W-byte slabs; work
//               item i = (slab, destination, run), claimed in order, so one
//               slab is stored to destination 0, then 1, ... and the DRAM
//               sees about one write stream at a time; the slab is read from
//               DRAM once and then hits L2
// GB/s = algorithmic (read + 8 x write) bytes / time; best of 5.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/bcast_l2_probe tools/bcast_l2_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) {                                                                \
      std::printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                         \
    }                                                                                       \
  } while (0)

namespace {

struct Dsts {
  char* d[8];
};

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
__device__ __forceinline__ void bstore(void* g, const void* s, uint32_t n, uint64_t pol) {
  if (pol)
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(g),
                 "r"(sa(s)), "r"(n), "l"(pol)
                 : "memory");
  else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(sa(s)), "r"(n)
                 : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* g, uint32_t n) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g), "r"(n) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// window: 0 = read the whole source; else wrap source offsets inside it.
// ahead: 0 = no prefetch; else prefetch the source `ahead` bytes past each run.
template <int S, int K>
__global__ void __launch_bounds__(32) bc_run(const char* src, Dsts dsts, size_t bytes, size_t run, unsigned int* ctr,
                                             size_t window, size_t ahead, int st_ef) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[S];
  if (threadIdx.x) return;
  uint64_t pol = 0;
  if (st_ef) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  for (int s = 0; s < S; ++s) mbar_init(&full[s]);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const size_t nruns = (bytes + run - 1) / run;
  size_t r = atomicAdd(ctr, 1u), off = 0;
  if (ahead && r < nruns && r * run + ahead < bytes) prefetch_l2(src + r * run + ahead, run);
  size_t issued = 0, done = 0;
  size_t cpos[S];
  for (;;) {
    while ((issued < S || issued - done < S - 1) && r < nruns) {
      if (issued >= S) wait_read1();
      const int s = issued % S;
      cpos[s] = r * run + off;
      mbar_expect(&full[s], K);
      bload(ring + s * K, src + (window ? cpos[s] % window : cpos[s]), K, &full[s]);
      ++issued;
      off += K;
      if (off >= run || r * run + off >= bytes) {
        off = 0;
        r = atomicAdd(ctr, 1u);
        if (ahead && r < nruns && r * run + ahead < bytes) prefetch_l2(src + r * run + ahead, run);
      }
    }
    if (done == issued) break;
    const int s = done % S;
    mbar_wait(&full[s], (done / S) & 1);
    for (int j = 0; j < 8; ++j) bstore(dsts.d[j] + cpos[s], ring + s * K, K, pol);
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

template <int S, int K>
__global__ void __launch_bounds__(32) bc_dmaj(const char* src, Dsts dsts, size_t bytes, size_t slab,
                                              unsigned int* ctr) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[S];
  if (threadIdx.x) return;
  for (int s = 0; s < S; ++s) mbar_init(&full[s]);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const size_t per_slab = slab / K;                       // runs per slab and destination
  const size_t nitems = bytes / slab * 8 * per_slab;      // bytes is a multiple of slab
  size_t issued = 0, done = 0;
  size_t pos[S];
  int dj[S];
  size_t i = atomicAdd(ctr, 1u);
  for (;;) {
    while ((issued < S || issued - done < S - 1) && i < nitems) {
      if (issued >= S) wait_read1();
      const int s = issued % S;
      const size_t sl = i / (8 * per_slab), rem = i % (8 * per_slab);
      dj[s] = static_cast<int>(rem / per_slab);
      pos[s] = sl * slab + (rem % per_slab) * K;
      mbar_expect(&full[s], K);
      bload(ring + s * K, src + pos[s], K, &full[s]);
      ++issued;
      i = atomicAdd(ctr, 1u);
    }
    if (done == issued) break;
    const int s = done % S;
    mbar_wait(&full[s], (done / S) & 1);
    bstore(dsts.d[dj[s]] + pos[s], ring + s * K, K, 0);
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

cudaEvent_t t0, t1;

template <class F>
float best_ms(F f) {
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
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

}  // namespace

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  const size_t G = size_t(1) << 30;
  // the product's geometry: replicas at a non-power-of-two stride
  const size_t sbo = 3 * G + G / 2;
  const size_t odd = sbo + (size_t(49) << 18) + 256;
  char* a = nullptr;
  CK(cudaMalloc(&a, 9 * odd));
  char* s = a + 8 * odd;
  Dsts d{};
  for (int j = 0; j < 8; ++j) d.d[j] = a + j * odd;
  CK(cudaMemset(s, 3, sbo));
  unsigned int* ctr = nullptr;
  CK(cudaMalloc(&ctr, 8));
  CK(cudaMemset(ctr, 0, 8));
  constexpr int S = 4, K = 16384;
  CK(cudaFuncSetAttribute(bc_run<S, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * K));
  const size_t run = 16384;
  auto go = [&](const char* name, int ctas, size_t window, size_t ahead, int st_ef) {
    const float ms = best_ms([&] { bc_run<S, K><<<ctas, 32, S * K>>>(s, d, sbo, run, ctr, window, ahead, st_ef); });
    std::printf("%-16s ctas=%-4d %8.3f ms %8.1f GB/s (writes alone %7.1f GB/s)\n", name, ctas, ms,
                9.0 * sbo / (ms * 1e6), 8.0 * sbo / (ms * 1e6));
    std::fflush(stdout);
  };
  for (int m : {1, 2}) {
    go("base", sms * m, 0, 0, 0);
    go("stEF", sms * m, 0, 0, 1);
    for (size_t w : {size_t(8) << 20, size_t(32) << 20}) {
      char nm[32];
      std::snprintf(nm, sizeof nm, "srcL2/%zuM", w >> 20);
      go(nm, sms * m, w, 0, 0);
    }
    for (size_t ah : {size_t(1) << 20, size_t(4) << 20, size_t(16) << 20, size_t(48) << 20}) {
      char nm[32];
      std::snprintf(nm, sizeof nm, "pf/%zuM", ah >> 20);
      go(nm, sms * m, 0, ah, 0);
    }
  }
  go("base", sms, 0, 0, 0);
  auto dmaj = [&](auto kern, int smem, const char* tag, std::initializer_list<int> mults) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int m : mults)
      for (size_t w : {size_t(1) << 20, size_t(2) << 20, size_t(4) << 20}) {
        const float ms = best_ms([&] { kern<<<sms * m, 32, smem>>>(s, d, sbo, w, ctr); });
        std::printf("dmaj%s/%zuM ctas=%-4d %8.3f ms %8.1f GB/s (writes alone %7.1f GB/s)\n", tag, w >> 20, sms * m, ms,
                    9.0 * sbo / (ms * 1e6), 8.0 * sbo / (ms * 1e6));
        std::fflush(stdout);
      }
  };
  dmaj(bc_dmaj<4, 16384>, 4 * 16384, "4x16k", {3});
  dmaj(bc_dmaj<4, 8192>, 4 * 8192, "4x8k", {4, 6});
  dmaj(bc_dmaj<2, 16384>, 2 * 16384, "2x16k", {4, 6});
  dmaj(bc_dmaj<3, 8192>, 3 * 8192, "3x8k", {6, 8});
  unsigned char h[2] = {0, 0};
  CK(cudaMemcpy(&h[0], d.d[7] + sbo - 1, 1, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&h[1], d.d[0], 1, cudaMemcpyDeviceToHost));
  std::printf("check %s\n", (h[0] == 3 && h[1] == 3) ? "ok" : "BAD");
  return 0;
}
