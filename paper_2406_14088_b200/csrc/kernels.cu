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

// L2-coherent load (bypasses L1): for relay sources that another GPU writes
// while this kernel runs (the .nc path above would be unsafe there).
__device__ __forceinline__ int4 ld_coherent(const int4* p) {
  int4 v;
  asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Relay wait: spin (acquire, system scope, bounded) until *flag >= epoch.
// Returns false on timeout (the caller counts it instead of hanging the GPU).
__device__ __forceinline__ bool wait_flag_geq(const uint32_t* flag, uint32_t epoch) {
  const uint64_t t0 = global_ns();
  while (true) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (static_cast<int32_t>(v - epoch) >= 0) return true;
    if (global_ns() - t0 > 20000000000ull) return false;
    __nanosleep(32);
  }
}

__device__ __forceinline__ void st_vec(int4* p, const int4& v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// NVLS multicast store: the NVSwitch replicates it into every member buffer.
// A plain bit move (.f32 is only the element type the v4 form requires).
__device__ __forceinline__ void st_multimem(int4* p, const int4& v) {
  asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
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
                                              uint32_t total, bool mc0, bool coherent) {
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
        const int4* p = src + static_cast<size_t>(row) * it.src_pitch + col;
        v[u] = coherent ? ld_coherent(p) : ld_stream(p);
        doff[u] = row * it.dst_pitch + col;  // < 2^32 units: checked on the host
      }
    }
    int j = 0;
    if (mc0) {  // one store through the multicast address reaches every group member
      int4* dst = reinterpret_cast<int4*>(dsts[0]);
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u)
        if (doff[u] != 0xffffffffu) st_multimem(dst + doff[u], v[u]);
      j = 1;
    }
    for (; j < ndst; ++j) {
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

// Dynamic work distribution: sched[0] is the next item, sched[1] counts
// CTAs that ran out of work; the last one resets both for the next launch.
__device__ __forceinline__ int grab_item(unsigned int* sched) { return static_cast<int>(atomicAdd(sched, 1u)); }

__device__ __forceinline__ void retire_cta(unsigned int* sched) {
  __threadfence();
  if (atomicAdd(sched + 1, 1u) == gridDim.x - 1) {
    atomicExch(sched, 0u);
    atomicExch(sched + 1, 0u);
  }
}

// sched[2] counts relay waits that timed out (reported by rr_exec_status).
__global__ void __launch_bounds__(kCopyThreads) rr_copy_kernel(const CopyItem* __restrict__ items, int n_items,
                                                               int fence_sys, unsigned int* sched, uint32_t epoch) {
  __shared__ CopyItem sh;
  __shared__ int cur;
  constexpr int kWords = sizeof(CopyItem) / 16;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) cur = grab_item(sched);
    __syncthreads();
    const int i = cur;
    if (i >= n_items) break;
    if (threadIdx.x < kWords)
      reinterpret_cast<int4*>(&sh)[threadIdx.x] = reinterpret_cast<const int4*>(items + i)[threadIdx.x];
    __syncthreads();
    if (sh.wait_flag) {  // relay: the previous GPU of the chain must have delivered this chunk
      if (threadIdx.x == 0 && !wait_flag_geq(reinterpret_cast<const uint32_t*>(sh.wait_flag), epoch))
        atomicAdd(sched + 2, 1u);
      __syncthreads();
    }
    CopyItem it;  // scalar fields only; the dst table stays in shared memory
    it.src = sh.src;
    it.row_units = sh.row_units;
    it.nrows = sh.nrows;
    it.src_pitch = sh.src_pitch;
    it.dst_pitch = sh.dst_pitch;
    it.inv_row = sh.inv_row;
    const int ndst = sh.ndst;
    const uint32_t total = it.row_units * it.nrows;
    if (sh.vec & kItemVec)
      copy_vec_item(it, sh.dst, ndst, total, (sh.vec & kItemMulticast0) != 0, sh.wait_flag != 0);
    else
      copy_elem_item(it, sh.dst, ndst, total);
    if (sh.signal_flag) {  // relay: release this chunk to the next GPU of the chain
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(sh.signal_flag), "r"(epoch) : "memory");
      }
    }
  }
  // Peer stores must be visible system-wide before a later barrier releases
  // them to the destination GPU.
  if (fence_sys) __threadfence_system();
  if (threadIdx.x == 0) retire_cta(sched);
}

// ---------------------------------------------------------------------------
// rr_bulk_kernel: the same work items, moved by the TMA engine. One elected
// thread per CTA streams pieces of each item through a ring of shared-memory
// stages: cp.async.bulk global->shared completes on a per-stage mbarrier,
// then one cp.async.bulk shared->global per destination (per row when the
// destination is strided) drains the stage. No data passes through
// registers, so one thread keeps ~S stages of loads and stores in flight.
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(smem_dst)),
               "l"(gmem_src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void bulk_store(void* gmem_dst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
               "r"(smem_addr(smem_src)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Full completion (writes performed, not only shared memory read) of all but
// the N most recent bulk groups.
template <int N>
__device__ __forceinline__ void bulk_wait_group() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Relay signal after the chunk's bulk stores completed: order them (async
// proxy) before the generic-proxy flag store, at system scope.
__device__ __forceinline__ void release_signal(uint64_t flag, uint32_t epoch) {
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
}

// One piece = up to `rows` rows of `row_bytes` (all 16-byte multiples).
struct Piece {
  uint64_t src;
  uint32_t rows, row_bytes, src_pitch, dst_pitch;  // bytes
  uint64_t dst_off;                                 // byte offset added to every dst base
  int item;
  bool last;  // the item's final piece (its relay signal follows it)
};

// Walks the items this CTA claims from the dynamic counter, in pieces of at
// most `cap` bytes.
struct PieceCursor {
  int item;
  uint32_t row, col;  // next row; next column byte offset inside the row
  bool waited;        // the current item's relay wait is satisfied
};

enum PieceStatus { kNoWork = 0, kPiece = 1, kBlocked = 2 };

// kBlocked: the next item waits on a relay flag and the caller still holds
// issued pieces. It must finish them (their signals may be what another GPU
// waits for) and call again with can_block before this CTA may spin.
__device__ __forceinline__ PieceStatus next_piece(const CopyItem* __restrict__ items, int n_items, PieceCursor& c,
                                                  uint32_t cap, Piece& p, unsigned int* sched, bool can_block,
                                                  uint32_t epoch) {
  while (c.item < n_items) {
    const CopyItem& it = items[c.item];
    const uint32_t row_bytes = it.row_units * 16u;
    const uint32_t sp = it.src_pitch * 16u, dp = it.dst_pitch * 16u;
    if (c.row < it.nrows) {
      if (it.wait_flag && !c.waited) {
        if (!can_block) return kBlocked;
        if (!wait_flag_geq(reinterpret_cast<const uint32_t*>(it.wait_flag), epoch)) atomicAdd(sched + 2, 1u);
        // the chunk was written by another GPU's generic-proxy stores; order
        // the TMA (async-proxy) reads of it after the acquire
        asm volatile("fence.proxy.async.global;" ::: "memory");
        c.waited = true;
      }
      p.item = c.item;
      if (row_bytes <= cap) {
        const uint32_t rows = min(it.nrows - c.row, max(1u, cap / row_bytes));
        p.src = it.src + static_cast<uint64_t>(c.row) * sp;
        p.dst_off = static_cast<uint64_t>(c.row) * dp;
        p.rows = rows;
        p.row_bytes = row_bytes;
        c.row += rows;
      } else {
        const uint32_t cols = min(row_bytes - c.col, cap);
        p.src = it.src + static_cast<uint64_t>(c.row) * sp + c.col;
        p.dst_off = static_cast<uint64_t>(c.row) * dp + c.col;
        p.rows = 1;
        p.row_bytes = cols;
        c.col += cols;
        if (c.col >= row_bytes) {
          c.col = 0;
          ++c.row;
        }
      }
      p.src_pitch = sp;
      p.dst_pitch = dp;
      p.last = c.row >= it.nrows;
      return kPiece;
    }
    c.item = grab_item(sched);
    c.row = c.col = 0;
    c.waited = false;
  }
  return kNoWork;
}

// Relay / overlapped fan-out items (wait_flag, signal_flag) run here too, so
// a flag-synchronised phase keeps the TMA ring's HBM efficiency. A CTA never
// spins on a wait while it holds issued pieces: it first drains its ring
// (stores, completion, signals), so every claimed push is finished by a CTA
// that cannot block on it, and the round ordering argument of build_items
// (exec_plan.cpp) carries over from the LDG/STG kernel.
template <int S, int STAGE>
__global__ void __launch_bounds__(32) rr_bulk_kernel(const CopyItem* __restrict__ items, int n_items,
                                                     int fence_sys, unsigned int* sched, uint32_t epoch) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[S];
  __shared__ Piece meta[S];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");

  PieceCursor ld{grab_item(sched), 0, 0, false};
  Piece p;
  auto issue_load = [&](int s) {
    meta[s] = p;
    const uint32_t bytes = p.rows * p.row_bytes;
    mbar_expect_tx(&full[s], bytes);
    uint8_t* buf = ring + s * STAGE;
    if (p.rows == 1 || p.src_pitch == p.row_bytes) {
      bulk_load(buf, reinterpret_cast<const void*>(p.src), bytes, &full[s]);
    } else {
      for (uint32_t r = 0; r < p.rows; ++r)
        bulk_load(buf + r * p.row_bytes, reinterpret_cast<const void*>(p.src + static_cast<uint64_t>(r) * p.src_pitch),
                  p.row_bytes, &full[s]);
    }
  };

  // Stage k % S holds piece k. Piece k may be loaded once the store group of
  // piece k - S has finished reading shared memory; keeping one committed
  // group in flight (wait_group.read 1) leaves S - 1 loads outstanding.
  int issued = 0, done = 0;
  uint64_t pending = 0;  // signal flag of a finished chunk not yet released
  for (;;) {
    PieceStatus st = kPiece;
    while (issued < S || issued - done < S - 1) {
      st = next_piece(items, n_items, ld, STAGE, p, sched, issued == done, epoch);
      if (st != kPiece) break;
      if (issued >= S) bulk_wait_read<1>();
      issue_load(issued % S);
      ++issued;
    }
    if (done == issued) {
      if (st == kNoWork) break;
      continue;  // blocked with an empty ring: the next call may spin
    }
    const int s = done % S;
    mbar_wait(&full[s], (done / S) & 1);
    const Piece q = meta[s];
    const CopyItem& it = items[q.item];
    const uint8_t* buf = ring + s * STAGE;
    const int ndst = it.ndst;
    for (int j = 0; j < ndst; ++j) {
      uint8_t* dst = reinterpret_cast<uint8_t*>(it.dst[j]) + q.dst_off;
      if (q.rows == 1 || q.dst_pitch == q.row_bytes) {
        bulk_store(dst, buf, q.rows * q.row_bytes);
      } else {
        for (uint32_t r = 0; r < q.rows; ++r)
          bulk_store(dst + static_cast<uint64_t>(r) * q.dst_pitch, buf + r * q.row_bytes, q.row_bytes);
      }
    }
    bulk_commit();
    ++done;
    // A finished chunk is released to the GPU that waits for it one piece
    // later: by now the store group before this one has usually landed, so
    // waiting for its completion costs little, whereas waiting for the group
    // just committed would stall the ring for a full NVLink round trip.
    if (pending) {
      bulk_wait_group<1>();
      release_signal(pending, epoch);
      pending = 0;
    }
    if (q.last && it.signal_flag) pending = it.signal_flag;
    if (pending && done == issued) {  // about to spin or exit: nothing may stay unreleased
      bulk_wait_all();
      release_signal(pending, epoch);
      pending = 0;
    }
  }
  bulk_wait_all();
  if (fence_sys) __threadfence_system();
  retire_cta(sched);
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

int launch_copy(const CopyItem* items, int n_items, int ctas, int fence_sys, void* stream, unsigned int* sched,
                uint32_t epoch) {
  if (n_items <= 0) return cudaSuccess;
  if (ctas > n_items) ctas = n_items;
  rr_copy_kernel<<<ctas, kCopyThreads, 0, static_cast<cudaStream_t>(stream)>>>(items, n_items, fence_sys, sched,
                                                                                epoch);
  return cudaGetLastError();
}

namespace {

template <int S, int STAGE>
int launch_bulk_t(const CopyItem* items, int n_items, int ctas, int fence_sys, void* stream, int* max_ctas,
                  unsigned int* sched, uint32_t epoch) {
  constexpr int kSmem = S * STAGE;
  cudaError_t e = cudaFuncSetAttribute(rr_bulk_kernel<S, STAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  if (e != cudaSuccess) return e;
  if (max_ctas) {
    int dev = 0, sms = 0, per_sm = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rr_bulk_kernel<S, STAGE>, 32, kSmem);
    if (e != cudaSuccess) return e;
    *max_ctas = per_sm * sms;
    return cudaSuccess;
  }
  if (n_items <= 0) return cudaSuccess;
  if (ctas > n_items) ctas = n_items;
  rr_bulk_kernel<S, STAGE><<<ctas, 32, kSmem, static_cast<cudaStream_t>(stream)>>>(items, n_items, fence_sys,
                                                                                        sched, epoch);
  return cudaGetLastError();
}

}  // namespace

// The two ring shapes the r01 sweeps kept (profiles/r01_sweep_kernels*.txt,
// r01_flag_kernel_sweep_n{2,4}.txt; the sweep variants live in tools/ history):
//   1: 4 x 16 KiB stages, 3 CTAs/SM — plain phases (96.9% of the HBM copy peak);
//   5: 3 x 16 KiB stages, 4 CTAs/SM — flag-synchronised phases, where more
//      resident CTAs keep NVLink busy while some spin on a flag.
int launch_bulk(int variant, const CopyItem* items, int n_items, int ctas, int fence_sys, void* stream,
                int* max_ctas, unsigned int* sched, uint32_t epoch) {
  switch (variant) {
    case 1: return launch_bulk_t<4, 16384>(items, n_items, ctas, fence_sys, stream, max_ctas, sched, epoch);
    case 5: return launch_bulk_t<3, 16384>(items, n_items, ctas, fence_sys, stream, max_ctas, sched, epoch);
    default: return cudaErrorInvalidValue;
  }
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
