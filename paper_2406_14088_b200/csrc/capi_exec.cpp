// C ABI, executor half (include/rr_realloc.h "execution"): builds the copy
// items of a lowered plan for one GPU (exec_plan.cpp), uploads them and
// launches the sm_100a kernels (kernels.cu) phase by phase, optionally
// pipelined behind a host->device onload.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <memory>
#include <vector>

#include "capi_internal.hpp"
#include "exec_plan.hpp"
#include "rr_internal.hpp"

using namespace rlplan;
using rr::capi::check_cuda;
using rr::capi::guarded;
using rr::capi::need;

namespace {
constexpr int64_t kDefaultChunk = int64_t{256} << 10;      // work-item size of large phases
constexpr int64_t kSmallPhaseBytes = int64_t{64} << 20;    // below: LDG/STG kernel (phase_kernel)
constexpr int64_t kMinSmallChunk = 4096;                   // 256 threads x one 16-byte load
// Copy-engine runs: a whole copy of >= 256 MiB over NVLink reaches 764-780
// GB/s against ~700-716 for SM stores, pairwise at 2 and 4 GPUs; at 64 MiB
// the engine's per-copy cost already eats the gain (profiles/r01_ce_probe_*).
constexpr int64_t kDefaultCeRunBytes = int64_t{256} << 20;

// Staged gather: each pushed piece is flagged by the copy stream itself
// (cuStreamWriteValue32, default flags: preceded by a system-wide memory
// barrier, so the piece's bytes are visible before the flag). No SM takes
// part, so a receiver's spinning unpack CTAs can never starve the signal that
// releases them. Resolved at run time like the multicast API (mcast.cpp): the
// library keeps no link dependency on libcuda.
using WriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

WriteValue32Fn write_value32() {
  static const WriteValue32Fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<WriteValue32Fn>(nullptr);
    }
    return reinterpret_cast<WriteValue32Fn>(p);
  }();
  return fn;
}

using WaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

// Copy-engine schedule: the copy stream itself waits until a flag reaches
// the launch epoch (cuStreamWaitValue32, GEQ: (int32)(*flag - epoch) >= 0),
// without an SM.
void wait_piece(cudaStream_t stream, const uint32_t* flag, uint32_t epoch) {
  static const WaitValue32Fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<WaitValue32Fn>(nullptr);
    }
    return reinterpret_cast<WaitValue32Fn>(p);
  }();
  if (fn == nullptr) rr::capi::raise(RR_EUNSUPPORTED, "cuStreamWaitValue32 unavailable (copy-engine schedule)");
  const CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), epoch,
                        CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) rr::capi::raise(RR_ECUDA, "cuStreamWaitValue32 (copy-engine schedule) failed: " + std::to_string(r));
}

void signal_piece(cudaStream_t stream, uint32_t* flag, uint32_t epoch) {
  const WriteValue32Fn fn = write_value32();
  if (fn == nullptr) rr::capi::raise(RR_EUNSUPPORTED, "cuStreamWriteValue32 unavailable (staged gather)");
  const CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), epoch,
                        CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) rr::capi::raise(RR_ECUDA, "cuStreamWriteValue32 (staged piece flag) failed: " + std::to_string(r));
}
}  // namespace

// ---------------------------------------------------------------------------
// Executor object
// ---------------------------------------------------------------------------

struct rr_exec {
  struct Phase {
    rr::CopyItem* d = nullptr;  // 16-byte (vec) items first, then 2-byte items
    int n = 0, n_vec = 0;
    int64_t read = 0, written = 0;
    bool flagged = false;  // relay / overlapped fan-out flags: one kernel runs the whole phase
  };
  int cuda_device = 0;
  Phase phase[2];  // [0] direct copies, [1] in-host fan-out from leader replicas
  int fence_sys = 0;
  int default_ctas = 0;
  // 0 = LDG/STG rr_copy_kernel, 1 / 5 = TMA bulk ring. Defaults
  // from the r01 sweeps: variant 1 (4 x 16 KiB stages, 3 CTAs/SM) for plain
  // phases, variant 5 (3 x 16 KiB, 4 CTAs/SM) for flag-synchronised ones,
  // where more resident CTAs keep NVLink busy while some spin on a flag
  // (profiles/r01_flag_kernel_sweep_n{2,4}.txt).
  int kernel = 1, flag_kernel = 5;
  // Plain phases that store fewer bytes than this take the LDG/STG kernel
  // unless a kernel was chosen explicitly: a small phase has few items, and
  // the bulk ring issues each item's (often narrow-row) stores from one
  // thread, whereas the LDG/STG kernel spreads an item over 256 threads
  // (tiny BASELINE config: 16 vs 39 us, profiles/r01_launch_latency_n1.json).
  bool kernel_explicit = false;
  int64_t small_phase_bytes = kSmallPhaseBytes;
  int bulk_ctas = 0, flag_bulk_ctas = 0;
  unsigned int* d_sched = nullptr;  // dynamic work counter (see retire_cta)
  int64_t wire_in = 0, wire_out = 0;  // bytes crossing into / out of this host
  uint32_t epoch = 0;                 // relay flag epoch, advanced by every phase-0 launch

  // Onload pipelining (rr_exec_enable_onload): phase-0 items regrouped into
  // segments by the last host->device chunk they read; segment s may start
  // once chunk s has landed.
  rr::ItemSet phase0_host;             // items + provenance as built
  std::vector<void*> src_bases;        // source buffer per plan device
  struct Segment {
    int offset = 0, n = 0, n_vec = 0;
  };
  std::vector<Segment> segments;       // [0] = no dependency, [1 + c] waits for chunk c
  rr::CopyItem* d_onload = nullptr;
  struct Chunk {
    int32_t device;
    int64_t offset, bytes;
  };
  std::vector<Chunk> chunks;
  std::vector<cudaEvent_t> events;

  // Copy-engine runs of phase 0 (rr::CeRun): issued on ce_stream, forked
  // from and joined back into the launching stream around the kernels.
  // A copy-engine submission: a contiguous run (height = depth = 1), or a
  // copy-engine transport copy (2D / 3D, rr::CeCopy).
  struct CeCopy {
    char* dst;
    const char* src;
    int64_t width, height, depth, src_pitch, dst_pitch, src_slice, dst_slice;
    DeviceId src_dev;  // source plan device and byte offsets in its shard (onload pipelining)
    int64_t src_off, src_end;
    uint32_t* flag = nullptr;  // copy-engine star: flagged on the receiving host after the copy
    uint32_t* wait = nullptr;  // schedule: wait (>= epoch) before the copy, on this host's array
    uint32_t* done = nullptr;  // schedule: raised after the copy (the next sender into its receiver)
    bool hard_wait = false;    // relay forward: `wait` is a data dependency (kept with an onload)
    int64_t bytes() const { return width * height * depth; }
  };
  std::vector<CeCopy> ce;
  int64_t ce_bytes = 0;
  // Staged gather, sender side: whole local source shards pushed piece by
  // piece into the other hosts' staging buffers, each piece followed by a
  // stream write (signal_piece) that flags it in the receiver's stage flag
  // array.
  struct StagePush {
    void* dst;
    const void* src;
    size_t bytes;      // 0: a round with nothing to send (it still passes the round token)
    uint32_t* flag;    // this piece's slot in the receiver's stage flag array (null when bytes == 0)
    DeviceId src_dev;  // source plan device and byte offset in its shard (onload pipelining)
    int64_t src_off;
    // Round alignment: the first push of round r waits until the previous
    // round's sender into the same receiver is done (`wait`, this host's
    // array); the last push of the round passes the token on (`done`).
    uint32_t* wait = nullptr;
    uint32_t* done = nullptr;
  };
  std::vector<StagePush> stage;
  int64_t stage_bytes = 0;
  // A staged executor's unpack kernel runs one CTA per SM unless the caller
  // picks a count: more CTAs only add HBM pressure and spinning against the
  // copy engines (profiles/r01_staged_sweep_n4.txt: 16.27 ms at 148 CTAs vs
  // 16.84 at 296 and 16.66 at 74, 7B tp8->dp8 forward, 4 GPUs).
  int stage_ctas = 0;
  // With an onload, the staged unpack runs from the start on its own stream
  // (and work counter) beside the per-chunk local copies.
  cudaStream_t unpack_stream = nullptr;
  cudaEvent_t unpack_fork = nullptr, unpack_join = nullptr;
  unsigned int* d_sched2 = nullptr;
  cudaStream_t ce_stream = nullptr;
  cudaEvent_t ce_fork = nullptr, ce_join = nullptr;

  rr_exec() = default;
  rr_exec(const rr_exec&) = delete;
  rr_exec& operator=(const rr_exec&) = delete;
  // Frees whatever was allocated, also when rr_exec_create_ex fails half way.
  ~rr_exec() {
    cudaSetDevice(cuda_device);
    for (auto& ph : phase)
      if (ph.d) cudaFree(ph.d);
    if (d_sched) cudaFree(d_sched);
    if (d_onload) cudaFree(d_onload);
    for (auto e : events) cudaEventDestroy(e);
    if (ce_fork) cudaEventDestroy(ce_fork);
    if (ce_join) cudaEventDestroy(ce_join);
    if (ce_stream) cudaStreamDestroy(ce_stream);
    if (unpack_fork) cudaEventDestroy(unpack_fork);
    if (unpack_join) cudaEventDestroy(unpack_join);
    if (unpack_stream) cudaStreamDestroy(unpack_stream);
    if (d_sched2) cudaFree(d_sched2);
  }
};

namespace {

// Host map for an executor: `local` plan devices form this host; without an
// explicit table every other device is its own host.
rr::HostMap host_map(const rr_plan* plan, int n_local, const int32_t* local, const int32_t* host_of) {
  const int n = plan->cluster.device_count();
  rr::HostMap hm;
  hm.host.resize(static_cast<size_t>(n));
  if (host_of) {
    for (int d = 0; d < n; ++d) hm.host[static_cast<size_t>(d)] = host_of[d];
    need(n_local > 0, "host_of needs at least one local device");
    need(local[0] >= 0 && local[0] < n, "local device out of range");
    hm.me = host_of[local[0]];
    for (int i = 0; i < n_local; ++i) {
      need(local[i] >= 0 && local[i] < n, "local device out of range");
      need(host_of[local[i]] == hm.me, "local devices must share one host");
    }
    return hm;
  }
  hm.hierarchical = false;
  for (int d = 0; d < n; ++d) hm.host[static_cast<size_t>(d)] = n + d;  // distinct remote hosts
  hm.me = -1;
  for (int i = 0; i < n_local; ++i) {
    need(local[i] >= 0 && local[i] < n, "local device out of range");
    hm.host[static_cast<size_t>(local[i])] = hm.me;
  }
  return hm;
}

void upload(const rr::ItemSet& set, rr_exec::Phase& ph) {
  ph.n = static_cast<int>(set.items.size());
  ph.n_vec = set.n_vec;
  ph.read = set.read;
  ph.written = set.written;
  ph.flagged = std::any_of(set.items.begin(), set.items.end(),
                           [](const rr::CopyItem& it) { return it.wait_flag || it.signal_flag; });
  if (set.items.empty()) return;
  const size_t bytes = set.items.size() * sizeof(rr::CopyItem);
  check_cuda(cudaMalloc(&ph.d, bytes), "cudaMalloc(items)");
  check_cuda(cudaMemcpy(ph.d, set.items.data(), bytes, cudaMemcpyHostToDevice), "upload items");
}

int phase_kernel(const rr_exec* ex, const rr_exec::Phase& ph) {
  if (ph.flagged) return ex->flag_kernel;
  if (!ex->kernel_explicit && ph.written < ex->small_phase_bytes) return 0;
  return ex->kernel;
}

void launch_phase(rr_exec* ex, const rr_exec::Phase& ph, void* stream, int ctas, unsigned int* sched = nullptr) {
  if (sched == nullptr) sched = ex->d_sched;
  check_cuda(cudaSetDevice(ex->cuda_device), "cudaSetDevice");
  if (ph.n == 0) return;
  const int kernel = phase_kernel(ex, ph);
  // A staged unpack spins on piece flags: it runs one CTA per SM on either
  // kernel, so it never fills the GPU (the flags themselves are raised by the
  // senders' copy streams, signal_piece, and need no SM here).
  const int ldst_ctas = ctas > 0 ? ctas : (ex->stage_ctas > 0 ? ex->stage_ctas : ex->default_ctas);
  if (kernel == 0) {
    check_cuda(rr::launch_copy(ph.d, ph.n, ldst_ctas, ex->fence_sys, stream, sched, ex->epoch), "rr_copy_kernel launch");
    return;
  }
  // Multicast and 2-byte items take the LDG/STG kernel, then the TMA bulk
  // kernel. A flag-synchronised phase is entirely in one of the two
  // (exec_plan.cpp build_items).
  if (ph.n > ph.n_vec)
    check_cuda(rr::launch_copy(ph.d + ph.n_vec, ph.n - ph.n_vec, ldst_ctas, ex->fence_sys, stream, sched, ex->epoch),
               "rr_copy_kernel launch (relay / multicast / 2-byte items)");
  if (ph.n_vec > 0)
    check_cuda(rr::launch_bulk(kernel, ph.d, ph.n_vec,
                               ctas > 0 ? ctas
                                        : (ex->stage_ctas > 0 ? ex->stage_ctas
                                                              : (ph.flagged ? ex->flag_bulk_ctas : ex->bulk_ctas)),
                               ex->fence_sys,
                               stream, nullptr, sched, ex->epoch),
               "rr_bulk_kernel launch");
}

// Work-item size of a plain phase when the caller left chunk_bytes at the
// default. Dynamic claiming balances the CTAs to within about one item, so
// the tail of a phase is one item's worth of work:
// - a small phase (LDG/STG kernel, phase_kernel) is latency-bound and lasts
//   as long as its largest item; with 256 KiB items the tiny BASELINE plan
//   had 78 items for 1184 resident CTAs. It is re-cut to about one item per
//   resident CTA (>= 4 KiB: 256 threads x one 16-byte load);
// - a larger phase gets at least kItemsPerBulkCta items per resident bulk CTA
//   (>= 32 KiB per item): a 256 MiB data-transfer phase had 1024 items for
//   444 CTAs, so its last wave ran a third full.
// Flag-synchronised phases keep the slot granularity every rank agrees on.
constexpr int64_t kItemsPerBulkCta = 16;
constexpr int64_t kMinBulkChunk = int64_t{32} << 10;
constexpr int64_t kWriteWindowMiB = 16;               // see refine_chunk
constexpr int64_t kMinWindowChunk = int64_t{16} << 10;  // one ring stage

rr::ItemSet refine_chunk(rr::ItemSet set, const std::vector<rr::Job>& jobs, int phase, const rr::HostMap& hm,
                         void* const* src_bufs, void* const* dst_bufs, int ldst_ctas, int bulk_ctas,
                         const std::vector<rr::CeRun>* ce) {
  if (set.items.empty()) return set;
  if (std::any_of(set.items.begin(), set.items.end(),
                  [](const rr::CopyItem& it) { return it.wait_flag || it.signal_flag; }))
    return set;
  int64_t chunk =
      set.written < kSmallPhaseBytes
          ? std::max<int64_t>(kMinSmallChunk, (set.read / std::max(1, ldst_ctas)) & ~int64_t{15})
          : std::max<int64_t>(kMinBulkChunk, (set.read / (kItemsPerBulkCta * std::max(1, bulk_ctas))) & ~int64_t{15});
  if (set.written >= kSmallPhaseBytes && !set.remote_stores) {
    // Write window (HBM phases): every resident CTA stores its current item
    // to each of the item's destinations, so CTAs x item x fan-out bytes are
    // being written at once. Keeping that near 16 MiB keeps the DRAM write
    // streams local: the 7B forward (a 1:8 broadcast) gets 16 KiB items, the
    // 1:1 back phase ~37 KiB; the default step is 1.9% faster than with
    // 256 KiB items (profiles/r02_window_sweep_n1.txt; 8 MiB starves the 1:1
    // phase, >= 64 MiB loses the gain). Phases with peer stores keep their
    // item size. RR_WRITE_WINDOW_MIB overrides it for sweeps (0 = off).
    const char* env = std::getenv("RR_WRITE_WINDOW_MIB");
    const int64_t window = (env ? std::atoll(env) : kWriteWindowMiB) << 20;
    const double fanout = set.read > 0 ? static_cast<double>(set.written) / static_cast<double>(set.read) : 1.0;
    const int64_t w = static_cast<int64_t>(static_cast<double>(window) / (std::max(1, bulk_ctas) * fanout)) & ~int64_t{15};
    if (window > 0) chunk = std::min(chunk, std::max(kMinWindowChunk, w));
  }
  if (chunk >= kDefaultChunk) return set;
  return rr::build_items(jobs, phase, hm, src_bufs, dst_bufs, chunk, ce);
}

// Copy-engine runs for a push executor: for every (local source, remote
// destination) pair of a plain phase-0 job, the maximal ranges where the two
// shard layouts coincide (rr::matching_runs), kept when >= min_bytes and when
// at least 98% of the range is bytes this pair is planned to move (so the
// engine does not carry data the destination gets elsewhere, e.g. locally).
std::vector<rr::CeRun> ce_runs(const rr_plan* plan, const std::vector<rr::Job>& jobs, const rr::HostMap& hm,
                               int64_t min_bytes) {
  std::map<std::pair<DeviceId, DeviceId>, std::vector<const rlplan::CopyRect*>> pairs;
  for (const auto& j : jobs) {
    if (j.phase != 0 || j.src_is_dst_buffer || j.multicast || j.relay_wait || j.relay_signal) continue;
    for (DeviceId d : j.dsts)
      if (hm.host[static_cast<size_t>(d)] != hm.me)
        for (const auto& r : j.op->rects) pairs[{j.src, d}].push_back(&r);
  }
  std::vector<rr::CeRun> out;
  for (const auto& [sd, rects] : pairs) {
    for (const auto& u : rr::matching_runs(plan->layout(0, sd.first), plan->layout(1, sd.second), sd.first,
                                           sd.second, min_bytes)) {
      int64_t planned = 0;
      for (const rlplan::CopyRect* r : rects)
        if (r->dst_off >= u.dst_off && rr::rect_dst_end(*r) <= u.dst_off + u.bytes) planned += rr::rect_bytes(*r);
      if (planned * 50 >= u.bytes * 49) out.push_back(u);
    }
  }
  return out;
}

void issue_copy(const rr_exec::CeCopy& c, cudaStream_t stream) {
  if (c.depth > 1) {
    cudaMemcpy3DParms p = {};
    p.srcPtr = make_cudaPitchedPtr(const_cast<char*>(c.src), static_cast<size_t>(c.src_pitch),
                                   static_cast<size_t>(c.width), static_cast<size_t>(c.src_slice / c.src_pitch));
    p.dstPtr = make_cudaPitchedPtr(c.dst, static_cast<size_t>(c.dst_pitch), static_cast<size_t>(c.width),
                                   static_cast<size_t>(c.dst_slice / c.dst_pitch));
    p.extent = make_cudaExtent(static_cast<size_t>(c.width), static_cast<size_t>(c.height),
                               static_cast<size_t>(c.depth));
    p.kind = cudaMemcpyDeviceToDevice;
    check_cuda(cudaMemcpy3DAsync(&p, stream), "copy-engine transport (3D)");
  } else if (c.height > 1) {
    check_cuda(cudaMemcpy2DAsync(c.dst, static_cast<size_t>(c.dst_pitch), c.src, static_cast<size_t>(c.src_pitch),
                                 static_cast<size_t>(c.width), static_cast<size_t>(c.height), cudaMemcpyDeviceToDevice,
                                 stream),
               "copy-engine transport (2D)");
  } else {
    check_cuda(cudaMemcpyAsync(c.dst, c.src, static_cast<size_t>(c.width), cudaMemcpyDeviceToDevice, stream),
               "copy-engine copy");
  }
}

// Copy-engine runs: start them on ce_stream once the work already queued on
// `after` (or, with an event, that event) is done; join them back into
// `into` so that whatever follows there (barrier, next phase) sees them.
void ce_issue(rr_exec* ex, cudaStream_t after, cudaEvent_t after_event = nullptr) {
  if (after_event == nullptr) {
    check_cuda(cudaEventRecord(ex->ce_fork, after), "cudaEventRecord(ce fork)");
    after_event = ex->ce_fork;
  }
  check_cuda(cudaStreamWaitEvent(ex->ce_stream, after_event, 0), "cudaStreamWaitEvent(ce fork)");
  for (const auto& c : ex->ce) {
    if (c.wait) wait_piece(ex->ce_stream, c.wait, ex->epoch);
    issue_copy(c, ex->ce_stream);
    if (c.flag) signal_piece(ex->ce_stream, c.flag, ex->epoch);
    if (c.done) signal_piece(ex->ce_stream, c.done, ex->epoch);
  }
  for (const auto& p : ex->stage) {
    if (p.wait) wait_piece(ex->ce_stream, p.wait, ex->epoch);
    if (p.bytes) {
      check_cuda(cudaMemcpyAsync(p.dst, p.src, p.bytes, cudaMemcpyDeviceToDevice, ex->ce_stream), "staged push");
      signal_piece(ex->ce_stream, p.flag, ex->epoch);
    }
    if (p.done) signal_piece(ex->ce_stream, p.done, ex->epoch);
  }
}

// Staged gather: the round tokens sit after every host's piece slots, at the
// same offset in every host's stage flag array (the largest piece count).
int64_t stage_sched_base(const rr_plan* plan, const rr::HostMap& hm, const std::vector<int64_t>& src_bytes) {
  std::vector<int> hosts(hm.host.begin(), hm.host.end());
  std::sort(hosts.begin(), hosts.end());
  hosts.erase(std::unique(hosts.begin(), hosts.end()), hosts.end());
  int64_t best = 0;
  for (int h : hosts) {
    int64_t k = 0;
    rr::stage_slots(plan->lowered, hm.host, h, src_bytes, hm.stage_chunk, &k);
    best = std::max(best, k);
  }
  return best;
}

// Largest row pitch a 2D / 3D copy accepts on this device.
int64_t max_pitch(int cuda_device) {
  int v = 0;
  check_cuda(cudaDeviceGetAttribute(&v, cudaDevAttrMaxPitch, cuda_device), "cudaDevAttrMaxPitch");
  return v;
}

// The first n uint32 of a flag array (mapped in this process) must be zero.
void require_zero_flags(const void* flags, int64_t n, const char* what) {
  if (flags == nullptr || n <= 0) return;
  std::vector<uint32_t> h(static_cast<size_t>(n));
  check_cuda(cudaMemcpy(h.data(), flags, h.size() * sizeof(uint32_t), cudaMemcpyDefault), "read flag array");
  if (std::any_of(h.begin(), h.end(), [](uint32_t v) { return v != 0; }))
    rr::capi::raise(RR_EINVAL, std::string(what) +
                                   ": flag array is not zero; zero it before every rr_exec_create_ex (one executor "
                                   "per array: epochs restart at 1 in a new executor)");
}

void ce_join(rr_exec* ex, cudaStream_t into) {
  check_cuda(cudaEventRecord(ex->ce_join, ex->ce_stream), "cudaEventRecord(ce join)");
  check_cuda(cudaStreamWaitEvent(into, ex->ce_join, 0), "cudaStreamWaitEvent(ce join)");
}

}  // namespace

rr_status rr_plan_work(const rr_plan* plan, int n_local, const int32_t* local, const int32_t* host_of, int mode,
                       int64_t* out6) {
  return guarded([&] {
    need(plan != nullptr && out6 != nullptr, "null plan/output");
    need(mode == 0 || mode == 1, "mode must be 0 (push) or 1 (pull)");
    const rr::HostMap hm = host_map(plan, n_local, local, host_of);
    const auto jobs = rr::build_jobs(plan->lowered, hm, mode);
    const auto a = rr::build_items(jobs, 0, hm, nullptr, nullptr, int64_t{1} << 30);
    const auto b = rr::build_items(jobs, 1, hm, nullptr, nullptr, int64_t{1} << 30);
    out6[0] = a.read;
    out6[1] = a.written;
    out6[2] = b.read;
    out6[3] = b.written;
    rr::host_wire_bytes(plan->lowered, hm, &out6[4], &out6[5]);
  });
}

rr_status rr_plan_stage_slots(const rr_plan* plan, const int32_t* host_of, int64_t chunk_bytes, int64_t* slots) {
  return guarded([&] {
    need(plan != nullptr && host_of != nullptr && slots != nullptr, "null plan/host table/output");
    need(chunk_bytes > 0, "chunk_bytes must be positive");
    const int n = plan->cluster.device_count();
    std::vector<int> host(host_of, host_of + n);
    std::vector<int64_t> src_bytes(static_cast<size_t>(n));
    for (int d = 0; d < n; ++d) src_bytes[static_cast<size_t>(d)] = plan->layout(0, d).bytes;
    int64_t best = 0;
    std::vector<int> hosts(host);
    std::sort(hosts.begin(), hosts.end());
    hosts.erase(std::unique(hosts.begin(), hosts.end()), hosts.end());
    for (int h : hosts) {
      int64_t k = 0;
      rr::stage_slots(plan->lowered, host, h, src_bytes, chunk_bytes, &k);
      best = std::max(best, k);
    }
    *slots = best + static_cast<int64_t>(hosts.size()) + 1;  // + the round tokens (stage_sched_base)
  });
}

rr_status rr_plan_ce_runs(const rr_plan* plan, int n_local, const int32_t* local, const int32_t* host_of,
                          int64_t min_run_bytes, int64_t* out5, int cap, int* n) {
  return guarded([&] {
    need(plan != nullptr && n != nullptr, "null plan/output");
    need(min_run_bytes > 0, "min_run_bytes must be positive");
    const rr::HostMap hm = host_map(plan, n_local, local, host_of);
    const auto jobs = rr::build_jobs(plan->lowered, hm, 0);
    const auto runs = ce_runs(plan, jobs, hm, min_run_bytes);
    *n = static_cast<int>(runs.size());
    if (out5 == nullptr) return;
    need(cap >= *n, "output table too small");
    for (size_t i = 0; i < runs.size(); ++i) {
      const auto& u = runs[i];
      int64_t* o = out5 + 5 * i;
      o[0] = u.src;
      o[1] = u.dst;
      o[2] = u.src_off;
      o[3] = u.dst_off;
      o[4] = u.bytes;
    }
  });
}

rr_status rr_plan_ce_copies(const rr_plan* plan, int n_local, const int32_t* local, const int32_t* host_of,
                            int64_t* out11, int cap, int* n) {
  return guarded([&] {
    need(plan != nullptr && n != nullptr, "null plan/output");
    rr::HostMap hm = host_map(plan, n_local, local, host_of);
    hm.ce_remote = true;
    const auto jobs = rr::build_jobs(plan->lowered, hm, 0);
    // host only: the pitch limit of B200 (cudaDevAttrMaxPitch = 2^31 - 1)
    const auto copies = rr::ce_transport_copies(jobs, hm, (int64_t{1} << 31) - 1);
    *n = static_cast<int>(copies.size());
    if (out11 == nullptr) return;
    need(cap >= *n, "output table too small");
    for (size_t i = 0; i < copies.size(); ++i) {
      const auto& c = copies[i];
      const int64_t v[11] = {c.src,   c.dst,       c.src_off,   c.dst_off,   c.width,    c.height,
                             c.depth, c.src_pitch, c.dst_pitch, c.src_slice, c.dst_slice};
      std::copy(v, v + 11, out11 + 11 * i);
    }
  });
}

rr_status rr_plan_ce_slots(const rr_plan* plan, const int32_t* host_of, int64_t* slots) {
  return guarded([&] {
    need(plan != nullptr && host_of != nullptr && slots != nullptr, "null plan/host table/output");
    rr::HostMap hm;
    for (int d = 0; d < plan->cluster.device_count(); ++d) hm.host.push_back(host_of[d]);
    std::vector<int> hosts(hm.host);
    std::sort(hosts.begin(), hosts.end());
    hosts.erase(std::unique(hosts.begin(), hosts.end()), hosts.end());
    int64_t best = 0;
    for (int relay = 0; relay < 2; ++relay)  // with and without relay chains (ce_transport 3 / 1-2)
      for (int h : hosts) {
        hm.me = h;
        hm.ce_relay = relay != 0;
        best = std::max(best, rr::ce_flag_slots(plan->lowered, hm, h, (int64_t{1} << 31) - 1));
      }
    *slots = best;
  });
}

rr_status rr_plan_ce_schedule(const rr_plan* plan, const int32_t* host_of, double* out6, int cap, int* n) {
  return guarded([&] {
    need(plan != nullptr && host_of != nullptr && n != nullptr, "null plan/host table/output");
    rr::HostMap hm;
    for (int d = 0; d < plan->cluster.device_count(); ++d) hm.host.push_back(host_of[d]);
    hm.me = hm.host.front();
    const int64_t mp = (int64_t{1} << 31) - 1;
    const auto sched = rr::ce_schedule(plan->lowered, hm, mp);
    *n = static_cast<int>(sched.size());
    if (out6 == nullptr) return;
    need(cap >= *n, "output table too small");
    std::map<int, std::vector<rr::CeCopy>> copies;
    for (size_t i = 0; i < sched.size(); ++i) {
      const auto& t = sched[i];
      if (!copies.count(t.sender)) copies[t.sender] = rr::ce_copies_of(plan->lowered, hm, t.sender, mp);
      int64_t bytes = 0;
      for (size_t k = t.first; k < t.first + t.count; ++k) bytes += copies[t.sender][k].bytes();
      const double v[6] = {static_cast<double>(t.sender), static_cast<double>(t.receiver), t.start, t.end,
                           t.wait_slot >= 0 ? 1.0 : 0.0, static_cast<double>(bytes)};
      std::copy(v, v + 6, out6 + 6 * i);
    }
  });
}

rr_status rr_exec_create(const rr_plan* plan, int cuda_device, int n_devices, void* const* src_bufs,
                         void* const* dst_bufs, int n_local, const int32_t* local, const int32_t* host_of,
                         int mode, int64_t chunk_bytes, rr_exec** out) {
  rr_exec_options opt;
  opt.mode = mode;
  opt.chunk_bytes = chunk_bytes;
  opt.host_of = host_of;
  opt.mc_bufs = nullptr;
  opt.relay_flags = nullptr;
  opt.relay_chain = 0;
  opt.overlap_fanout = 0;
  opt.ce_min_run_bytes = 0;
  opt.stage_chunk_bytes = 0;
  opt.n_hosts = 0;
  opt.stage_remote = nullptr;
  opt.stage_flags = nullptr;
  opt.ce_transport = 0;
  opt.ce_flags = nullptr;
  return rr_exec_create_ex(plan, cuda_device, n_devices, src_bufs, dst_bufs, n_local, local, &opt, out);
}

rr_status rr_exec_create_ex(const rr_plan* plan, int cuda_device, int n_devices, void* const* src_bufs,
                            void* const* dst_bufs, int n_local, const int32_t* local,
                            const rr_exec_options* options, rr_exec** out) {
  return guarded([&] {
    need(plan != nullptr && out != nullptr && options != nullptr, "null plan/options/output");
    const int mode = options->mode;
    int64_t chunk_bytes = options->chunk_bytes;
    need(mode == 0 || mode == 1, "mode must be 0 (push) or 1 (pull)");
    need(n_devices >= plan->cluster.device_count(), "buffer tables must cover every cluster device");
    if (chunk_bytes <= 0) chunk_bytes = kDefaultChunk;
    need(chunk_bytes >= 16, "chunk_bytes too small");
    rr::HostMap hm = host_map(plan, n_local, local, options->host_of);
    if (options->mc_bufs) {
      need(options->host_of != nullptr, "multicast needs a host_of table");
      need(mode == 0, "multicast is a push-mode path");
      hm.mc.resize(hm.host.size());
      for (size_t d = 0; d < hm.mc.size(); ++d) hm.mc[d] = reinterpret_cast<uint64_t>(options->mc_bufs[d]);
    }
    hm.relay_chunk = chunk_bytes;
    if (options->relay_flags) {
      need(options->host_of != nullptr && mode == 0, "relay needs a host_of table and push mode");
      hm.relay_flags.resize(hm.host.size());
      for (size_t d = 0; d < hm.relay_flags.size(); ++d)
        hm.relay_flags[d] = reinterpret_cast<uint64_t>(options->relay_flags[d]);
      hm.relay_chain = options->relay_chain != 0;
      hm.relay_star = options->overlap_fanout != 0;
    }
    std::vector<int64_t> src_bytes(static_cast<size_t>(plan->cluster.device_count()), 0);
    const bool staged = options->stage_chunk_bytes > 0;
    int64_t n_stage_slots = 0;
    if (staged) {
      need(mode == 1 && options->host_of != nullptr, "a staged gather runs in pull mode with a host_of table");
      need(options->stage_flags != nullptr && options->stage_remote != nullptr && options->n_hosts > 0,
           "staged gather needs stage_flags, stage_remote and n_hosts");
      need(options->relay_flags == nullptr && options->mc_bufs == nullptr, "staged gather excludes relay/multicast");
      for (size_t d = 0; d < hm.host.size(); ++d) {
        need(hm.host[d] >= 0 && hm.host[d] < options->n_hosts, "host ids must lie in 0..n_hosts-1");
        src_bytes[d] = plan->layout(0, static_cast<DeviceId>(d)).bytes;
      }
      hm.stage_chunk = options->stage_chunk_bytes;
      hm.stage_slot0 = rr::stage_slots(plan->lowered, hm.host, hm.me, src_bytes, hm.stage_chunk, &n_stage_slots);
      hm.stage_flags = reinterpret_cast<uint64_t>(options->stage_flags[hm.me]);
      need(n_stage_slots == 0 || hm.stage_flags != 0, "missing this host's stage flag array");
    }
    if (options->ce_transport) {
      need(mode == 0, "copy-engine transport is a push-mode path");
      need(!staged && options->mc_bufs == nullptr, "copy-engine transport excludes the staged gather and multicast");
      hm.ce_remote = true;
      hm.ce_hybrid = options->ce_transport == 2;
      hm.ce_relay = options->ce_transport == 3;
      need(options->ce_transport >= 1 && options->ce_transport <= 3,
           "ce_transport must be 0, 1, 2 (hybrid) or 3 (with relay chains)");
      need(!hm.ce_relay || options->ce_flags != nullptr, "the copy-engine relay needs ce_flags");
      need(!(hm.ce_hybrid && options->overlap_fanout), "the hybrid copy-engine transport excludes the star");
      need(options->relay_flags == nullptr, "copy-engine transport excludes relay flags");
      if (options->ce_flags) {
        need(options->host_of != nullptr && options->n_hosts > 0, "copy flags need host_of and n_hosts");
        for (size_t d = 0; d < hm.host.size(); ++d)
          need(hm.host[d] >= 0 && hm.host[d] < options->n_hosts, "host ids must lie in 0..n_hosts-1");
        hm.ce_flags = reinterpret_cast<uint64_t>(options->ce_flags[hm.me]);
        hm.ce_star = options->overlap_fanout != 0;  // fan-out on per-copy flags inside phase 0
      } else {
        need(options->overlap_fanout == 0, "the copy-engine star (overlap_fanout) needs ce_flags");
      }
    }
    check_cuda(cudaSetDevice(cuda_device), "cudaSetDevice");
    int per_sm = 0, sms = 0;
    check_cuda(rr::copy_max_ctas(&per_sm, &sms), "occupancy query");
    const auto jobs = rr::build_jobs(plan->lowered, hm, mode);
    if (hm.ce_hybrid)  // the rects the SM kernel keeps: known before the items are built
      rr::ce_transport_copies(jobs, hm, max_pitch(cuda_device), &hm.ce_sm_rects);
    const int64_t ce_min = options->ce_min_run_bytes == 0 ? kDefaultCeRunBytes : options->ce_min_run_bytes;
    const std::vector<rr::CeRun> runs =
        (mode == 0 && ce_min > 0 && src_bufs && dst_bufs && !hm.ce_remote) ? ce_runs(plan, jobs, hm, ce_min)
                                                                           : std::vector<rr::CeRun>{};
    std::vector<rr::CeCopy> transport;
    std::vector<int64_t> send_slots;
    std::vector<rr::CeTransfer> schedule;  // this host's transfers, issue order (with ce_flags)
    rr::CeSlotMap slot_map;
    int64_t n_ce_slots = 0;
    if (hm.ce_remote) {
      need(src_bufs != nullptr && dst_bufs != nullptr, "copy-engine transport needs buffer tables");
      const int64_t mp = max_pitch(cuda_device);
      transport = rr::ce_transport_copies(jobs, hm, mp);
      if (hm.ce_star) {
        send_slots = rr::ce_send_slots(plan->lowered, hm, transport, mp);
        const auto flagged = rr::star_flagged(transport, hm);
        for (size_t k = 0; k < send_slots.size(); ++k)
          if (!flagged[k]) send_slots[k] = -1;  // inside a flag group: no write after this copy
        slot_map = rr::ce_slot_map(plan->lowered, hm, hm.me, mp);
      }
      if (options->ce_flags) {
        for (const auto& t : rr::ce_schedule(plan->lowered, hm, mp))
          if (t.sender == hm.me) schedule.push_back(t);
        n_ce_slots = rr::ce_flag_slots(plan->lowered, hm, hm.me, mp);
        need(n_ce_slots == 0 || hm.ce_flags != 0, "missing this host's copy flag array");
      }
    }
    // copy-engine relay: ops, pieces, and this host's relay slot lookup
    std::vector<rr::CeRelayOp> relay_ops;
    std::map<int, int64_t> relay_base;  // per host: first relay slot in its flag array
    rr::RelaySlotFn relay_slot_fn;
    if (hm.ce_relay) {
      const int64_t mp = max_pitch(cuda_device);
      relay_ops = rr::ce_relay_ops(plan->lowered, hm);
      for (int h : std::set<int>(hm.host.begin(), hm.host.end())) relay_base[h] = rr::ce_relay_base(plan->lowered, hm, h, mp);
      const int64_t mine = relay_base[hm.me];
      relay_slot_fn = [&relay_ops, mine](const LoweredOp* op, int64_t byte) -> int64_t {
        for (const auto& r : relay_ops) {
          if (r.op != op) continue;
          for (size_t k = 0; k < r.pieces.size(); ++k) {
            const auto& p = r.pieces[k];
            int64_t rel = byte - p.dst_off;
            if (rel < 0) continue;
            if (p.height > 1) {
              const int64_t y = rel / p.dst_pitch;
              if (y >= p.height) continue;
              rel -= y * p.dst_pitch;
            }
            if (rel < p.width) return mine + r.slot0 + static_cast<int64_t>(k);
          }
        }
        return -1;
      };
    }
    auto a = rr::build_items(jobs, 0, hm, src_bufs, dst_bufs, chunk_bytes, &runs, hm.ce_star ? &slot_map : nullptr,
                             hm.ce_relay ? &relay_slot_fn : nullptr);
    auto b = rr::build_items(jobs, 1, hm, src_bufs, dst_bufs, chunk_bytes);
    if (options->chunk_bytes <= 0) {
      int bulk_ctas = 0;
      check_cuda(rr::launch_bulk(1, nullptr, 0, 0, 0, nullptr, &bulk_ctas, nullptr), "bulk occupancy");
      const int ldst_ctas = std::max(1, per_sm) * sms;
      a = refine_chunk(std::move(a), jobs, 0, hm, src_bufs, dst_bufs, ldst_ctas, bulk_ctas, &runs);
      b = refine_chunk(std::move(b), jobs, 1, hm, src_bufs, dst_bufs, ldst_ctas, bulk_ctas, nullptr);
    }

    // Flag arrays compare against a per-executor epoch that starts at 1, so an
    // array carrying values of an earlier executor would release waits before
    // their data lands. The array this host waits on must therefore be fresh
    // (zeroed) and owned by this executor alone (include/rr_realloc.h).
    if (options->relay_flags && !hm.relay_flags.empty()) {
      const int64_t n_relay = rr::relay_slots(plan->lowered, hm);
      require_zero_flags(options->relay_flags[local[0]], n_relay, "relay_flags");
    }
    if (staged) {
      std::vector<int> hs(hm.host.begin(), hm.host.end());
      std::sort(hs.begin(), hs.end());
      hs.erase(std::unique(hs.begin(), hs.end()), hs.end());
      require_zero_flags(options->stage_flags[hm.me],
                         std::max(n_stage_slots, stage_sched_base(plan, hm, src_bytes) + static_cast<int64_t>(hs.size()) + 1),
                         "stage_flags");
    }
    if (hm.ce_remote && options->ce_flags) require_zero_flags(options->ce_flags[hm.me], n_ce_slots, "ce_flags");

    auto ex = std::make_unique<rr_exec>();
    ex->cuda_device = cuda_device;
    // Remote accesses (peer stores, or peer loads in pull mode) must be
    // visible system-wide before the following barrier releases them.
    int64_t win = 0, wout = 0;
    rr::host_wire_bytes(plan->lowered, hm, &win, &wout);
    ex->fence_sys = (a.remote_stores || win || wout) ? 1 : 0;
    ex->wire_in = win;
    ex->wire_out = wout;
    ex->default_ctas = std::max(1, per_sm) * sms;
    upload(a, ex->phase[0]);
    upload(b, ex->phase[1]);
    for (const auto& u : runs) {
      ex->ce.push_back({static_cast<char*>(dst_bufs[u.dst]) + u.dst_off,
                        static_cast<const char*>(src_bufs[u.src]) + u.src_off, u.bytes, 1, 1, u.bytes, u.bytes, 0, 0,
                        u.src, u.src_off, u.src_off + u.bytes});
      ex->ce_bytes += u.bytes;
    }
    auto host_flags = [&](int h) {
      auto* arr = static_cast<uint32_t*>(options->ce_flags[h]);
      need(arr != nullptr, "missing a host's copy flag array");
      return arr;
    };
    auto push_copy = [&](size_t k, uint32_t* wait, uint32_t* done) {
      const auto& c = transport[k];
      need(dst_bufs[c.dst] != nullptr && src_bufs[c.src] != nullptr, "missing a copy-engine transport buffer");
      uint32_t* flag = hm.ce_star && send_slots[k] >= 0 ? host_flags(hm.host[static_cast<size_t>(c.dst)]) + send_slots[k]
                                                         : nullptr;
      ex->ce.push_back({static_cast<char*>(dst_bufs[c.dst]) + c.dst_off,
                        static_cast<const char*>(src_bufs[c.src]) + c.src_off, c.width, c.height, c.depth,
                        c.src_pitch, c.dst_pitch, c.src_slice, c.dst_slice, c.src, c.src_off, c.src_end(), flag,
                        wait, done});
      ex->ce_bytes += c.bytes();
    };
    // Copy-engine relay actions first, in (op, piece) order on every host:
    // a forward depends only on the same piece's previous hop, which every
    // other stream issues after strictly earlier pieces only, so no cycle;
    // the transport copies (their schedule waits point only to transport
    // copies) follow.
    for (const auto& r : relay_ops) {
      const LoweredOp& op = *r.op;
      const auto pos = std::find(r.chain.begin(), r.chain.end(), hm.me) - r.chain.begin();
      const bool sender = r.src_host == hm.me;
      const bool forwarder = pos + 1 < static_cast<std::ptrdiff_t>(r.chain.size());
      if (!sender && !forwarder) continue;
      const size_t next = sender ? 0 : static_cast<size_t>(pos) + 1;
      const int to_host = r.chain[next];
      for (size_t k = 0; k < r.pieces.size(); ++k) {
        const auto& p = r.pieces[k];
        const int64_t slot = r.slot0 + static_cast<int64_t>(k);
        rr_exec::CeCopy c{};
        c.dst = static_cast<char*>(dst_bufs[r.leader[next]]) + p.dst_off;
        c.width = p.width;
        c.height = p.height;
        c.depth = 1;
        c.dst_pitch = p.dst_pitch ? p.dst_pitch : p.width;
        c.src_slice = c.dst_slice = 0;
        c.flag = host_flags(to_host) + relay_base.at(to_host) + slot;
        if (sender) {
          need(src_bufs[op.src] != nullptr, "missing a relay source buffer");
          c.src = static_cast<const char*>(src_bufs[op.src]) + p.src_off;
          c.src_pitch = p.src_pitch ? p.src_pitch : p.width;
          c.src_dev = op.src;
          c.src_off = p.src_off;
          c.src_end = p.src_off + (p.height - 1) * c.src_pitch + p.width;
        } else {
          c.src = static_cast<const char*>(dst_bufs[r.leader[static_cast<size_t>(pos)]]) + p.dst_off;
          c.src_pitch = c.dst_pitch;
          c.src_dev = -1;  // this host's leader replica, not an onloaded source
          c.wait = host_flags(hm.me) + relay_base.at(hm.me) + slot;
          c.hard_wait = true;
        }
        need(c.dst != nullptr && c.src != nullptr, "missing a relay leader buffer");
        ex->ce.push_back(c);
        ex->ce_bytes += c.bytes();
      }
    }
    if (!schedule.empty()) {
      // scheduled issue order: each transfer waits for the previous one into
      // its receiver (if another host sent it) and releases the next
      size_t issued = 0;
      for (const auto& t : schedule) {
        for (size_t k = t.first; k < t.first + t.count; ++k) {
          uint32_t* wait = (k == t.first && t.wait_slot >= 0) ? host_flags(hm.me) + t.wait_slot : nullptr;
          uint32_t* done = (k + 1 == t.first + t.count && t.signal_host >= 0)
                               ? host_flags(t.signal_host) + t.signal_slot : nullptr;
          push_copy(k, wait, done);
          ++issued;
        }
      }
      need(issued == transport.size(), "copy-engine schedule does not cover every transport copy");
    } else {
      for (size_t k = 0; k < transport.size(); ++k) push_copy(k, nullptr, nullptr);
    }
    if (staged) {
      ex->stage_ctas = sms;
      check_cuda(cudaStreamCreateWithFlags(&ex->unpack_stream, cudaStreamNonBlocking), "cudaStreamCreate");
      check_cuda(cudaEventCreateWithFlags(&ex->unpack_fork, cudaEventDisableTiming), "cudaEventCreate");
      check_cuda(cudaEventCreateWithFlags(&ex->unpack_join, cudaEventDisableTiming), "cudaEventCreate");
      check_cuda(cudaMalloc(&ex->d_sched2, 4 * sizeof(unsigned int)), "cudaMalloc(sched)");
      check_cuda(cudaMemset(ex->d_sched2, 0, 4 * sizeof(unsigned int)), "cudaMemset(sched)");
      // Sender side: round r = 1..H-1 pushes to the host r places after
      // this one (the receiver's arrival order, rr::stage_sources).
      std::vector<int> hosts(hm.host.begin(), hm.host.end());
      std::sort(hosts.begin(), hosts.end());
      hosts.erase(std::unique(hosts.begin(), hosts.end()), hosts.end());
      const int H = static_cast<int>(hosts.size());
      const int pos = static_cast<int>(std::find(hosts.begin(), hosts.end(), hm.me) - hosts.begin());
      // Rounds stay aligned without a barrier: the round-r push into host h
      // waits for the round-(r-1) sender into h (the host one place after
      // this one) to finish, which raises slot sched_base + r in this
      // host's stage flag array; after its own round r this host raises slot
      // sched_base + r + 1 in the array of the host one place before it (the
      // round-(r+1) sender into h). Waits point only to the previous round:
      // no cycle. Unaligned, a sender whose round ran short pushed into a
      // receiver still taking the previous round's sender.
      const int64_t sched_base = stage_sched_base(plan, hm, src_bytes);
      const int prev_host = hosts[static_cast<size_t>((pos + H - 1) % H)];
      auto* my_flags = static_cast<uint32_t*>(options->stage_flags[hm.me]);
      auto* prev_flags = static_cast<uint32_t*>(options->stage_flags[prev_host]);
      need(my_flags != nullptr && prev_flags != nullptr, "missing a stage flag array");
      for (int r = 1; r < H; ++r) {
        const int h = hosts[static_cast<size_t>((pos + r) % H)];
        int64_t n_slots = 0;
        const auto slot0 = rr::stage_slots(plan->lowered, hm.host, h, src_bytes, hm.stage_chunk, &n_slots);
        const size_t first = ex->stage.size();
        for (DeviceId sdev : rr::stage_sources(plan->lowered, hm.host, h)) {
          if (hm.host[static_cast<size_t>(sdev)] != hm.me) continue;
          void* remote = options->stage_remote[static_cast<size_t>(sdev) * options->n_hosts + h];
          auto* flags = static_cast<uint32_t*>(options->stage_flags[h]);
          need(remote != nullptr && flags != nullptr, "missing a receiver's staging buffer or flag array");
          need(src_bufs != nullptr && src_bufs[sdev] != nullptr, "missing a staged source buffer");
          const int64_t total = src_bytes[static_cast<size_t>(sdev)];
          for (int64_t off = 0, c = 0; off < total; off += hm.stage_chunk, ++c) {
            const int64_t nb = std::min(hm.stage_chunk, total - off);
            ex->stage.push_back({static_cast<char*>(remote) + off, static_cast<const char*>(src_bufs[sdev]) + off,
                                 static_cast<size_t>(nb), flags + slot0[static_cast<size_t>(sdev)] + c, sdev, off});
            ex->stage_bytes += nb;
          }
        }
        if (ex->stage.size() == first)  // nothing for h this round: the token still passes
          ex->stage.push_back({nullptr, nullptr, 0, nullptr, -1, 0});
        if (r > 1) ex->stage[first].wait = my_flags + sched_base + r;
        if (r + 1 < H) ex->stage.back().done = prev_flags + sched_base + r + 1;
      }
    }
    if (!ex->ce.empty() || !ex->stage.empty()) {
      check_cuda(cudaStreamCreateWithFlags(&ex->ce_stream, cudaStreamNonBlocking), "cudaStreamCreate");
      check_cuda(cudaEventCreateWithFlags(&ex->ce_fork, cudaEventDisableTiming), "cudaEventCreate");
      check_cuda(cudaEventCreateWithFlags(&ex->ce_join, cudaEventDisableTiming), "cudaEventCreate");
    }
    ex->phase0_host = a;
    ex->src_bases.assign(static_cast<size_t>(n_devices), nullptr);
    for (int d = 0; d < n_devices; ++d) ex->src_bases[static_cast<size_t>(d)] = src_bufs ? src_bufs[d] : nullptr;
    check_cuda(cudaMalloc(&ex->d_sched, 4 * sizeof(unsigned int)), "cudaMalloc(sched)");
    check_cuda(cudaMemset(ex->d_sched, 0, 4 * sizeof(unsigned int)), "cudaMemset(sched)");
    check_cuda(rr::launch_bulk(ex->kernel, nullptr, 0, 0, 0, nullptr, &ex->bulk_ctas, nullptr), "bulk occupancy");
    check_cuda(rr::launch_bulk(ex->flag_kernel, nullptr, 0, 0, 0, nullptr, &ex->flag_bulk_ctas, nullptr),
               "bulk occupancy");
    *out = ex.release();
  });
}

rr_status rr_exec_launch(rr_exec* ex, void* stream, int ctas) {
  return guarded([&] {
    need(ex != nullptr, "null executor");
    ++ex->epoch;  // every rank launches phase 0 the same number of times
    auto st = static_cast<cudaStream_t>(stream);
    check_cuda(cudaSetDevice(ex->cuda_device), "cudaSetDevice");
    const bool side = !ex->ce.empty() || !ex->stage.empty();
    if (side) ce_issue(ex, st);
    launch_phase(ex, ex->phase[0], stream, ctas);
    if (side) ce_join(ex, st);
  });
}

rr_status rr_exec_kernel_count(const rr_exec* ex, int* phase0, int* phase1) {
  return guarded([&] {
    need(ex != nullptr, "null executor");
    auto count = [&](const rr_exec::Phase& ph) {
      if (ph.n == 0) return 0;
      if (phase_kernel(ex, ph) == 0) return 1;
      return (ph.n > ph.n_vec ? 1 : 0) + (ph.n_vec > 0 ? 1 : 0);
    };
    *phase0 = count(ex->phase[0]);
    *phase1 = count(ex->phase[1]);
  });
}

rr_status rr_exec_phase_kernels(const rr_exec* ex, int phase, int* ldst, int* bulk) {
  return guarded([&] {
    need(ex != nullptr && ldst != nullptr && bulk != nullptr, "null executor/output");
    need(phase == 0 || phase == 1, "phase must be 0 or 1");
    const auto& ph = ex->phase[phase];
    *ldst = 0;
    *bulk = 0;
    if (ph.n == 0) return;
    const int kernel = phase_kernel(ex, ph);
    if (kernel == 0) {
      *ldst = 1;
      return;
    }
    *ldst = ph.n > ph.n_vec ? 1 : 0;
    *bulk = ph.n_vec > 0 ? kernel : 0;
  });
}

rr_status rr_exec_ce_runs(const rr_exec* ex, int* n_runs, int64_t* bytes) {
  return guarded([&] {
    need(ex != nullptr && n_runs != nullptr && bytes != nullptr, "null executor/output");
    *n_runs = static_cast<int>(ex->ce.size());
    *bytes = ex->ce_bytes;
  });
}

rr_status rr_exec_stage_pushes(const rr_exec* ex, int* n_pushes, int64_t* bytes) {
  return guarded([&] {
    need(ex != nullptr && n_pushes != nullptr && bytes != nullptr, "null executor/output");
    *n_pushes = static_cast<int>(ex->stage.size());
    *bytes = ex->stage_bytes;
  });
}

rr_status rr_exec_relay_timeouts(rr_exec* ex, int64_t* timeouts) {
  return guarded([&] {
    need(ex != nullptr, "null executor");
    check_cuda(cudaSetDevice(ex->cuda_device), "cudaSetDevice");
    unsigned int h[4];
    check_cuda(cudaMemcpy(h, ex->d_sched, sizeof(h), cudaMemcpyDeviceToHost), "read relay status");
    *timeouts = h[2];
    if (ex->d_sched2) {
      check_cuda(cudaMemcpy(h, ex->d_sched2, sizeof(h), cudaMemcpyDeviceToHost), "read relay status");
      *timeouts += h[2];
    }
  });
}

rr_status rr_plan_relay_slots(const rr_plan* plan, const int32_t* host_of, int64_t chunk_bytes, int relay_chain,
                              int overlap_fanout, int64_t* slots) {
  return guarded([&] {
    need(plan != nullptr && host_of != nullptr, "null plan/host table");
    rr::HostMap hm;
    for (int d = 0; d < plan->cluster.device_count(); ++d) hm.host.push_back(host_of[d]);
    hm.relay_chunk = chunk_bytes > 0 ? chunk_bytes : kDefaultChunk;
    hm.relay_chain = relay_chain != 0;
    hm.relay_star = overlap_fanout != 0;
    *slots = rr::relay_slots(plan->lowered, hm);
  });
}

rr_status rr_exec_launch_fanout(rr_exec* ex, void* stream, int ctas) {
  return guarded([&] {
    need(ex != nullptr, "null executor");
    launch_phase(ex, ex->phase[1], stream, ctas);
  });
}

namespace {

void select_kernel(rr_exec* ex, int kernel, int* slot, int* slot_ctas) {
  need(ex != nullptr, "null executor");
  need(rr::valid_kernel(kernel), "unknown copy kernel (0 LDG/STG, 1 or 5 TMA bulk ring)");
  *slot = kernel;
  if (kernel > 0) {
    check_cuda(cudaSetDevice(ex->cuda_device), "cudaSetDevice");
    check_cuda(rr::launch_bulk(kernel, nullptr, 0, 0, 0, nullptr, slot_ctas, nullptr), "bulk occupancy");
  }
}

}  // namespace

rr_status rr_exec_set_kernel(rr_exec* ex, int kernel) {
  return guarded([&] {
    select_kernel(ex, kernel, &ex->kernel, &ex->bulk_ctas);
    ex->kernel_explicit = true;
  });
}

rr_status rr_exec_set_small_phase_bytes(rr_exec* ex, int64_t bytes) {
  return guarded([&] {
    need(ex != nullptr && bytes >= 0, "null executor or negative size");
    ex->small_phase_bytes = bytes;
  });
}

rr_status rr_exec_set_flag_kernel(rr_exec* ex, int kernel) {
  return guarded([&] { select_kernel(ex, kernel, &ex->flag_kernel, &ex->flag_bulk_ctas); });
}

rr_status rr_exec_stats(const rr_exec* ex, int phase, int64_t* items, int64_t* written, int64_t* read) {
  return guarded([&] {
    need(ex != nullptr, "null executor");
    need(phase == 0 || phase == 1, "phase must be 0 or 1");
    const auto& ph = ex->phase[phase];
    *items = ph.n;
    *written = ph.written + (phase == 0 ? ex->ce_bytes : 0);
    *read = ph.read + (phase == 0 ? ex->ce_bytes : 0);
  });
}

rr_status rr_exec_wire(const rr_exec* ex, int64_t* wire_in, int64_t* wire_out) {
  return guarded([&] {
    need(ex != nullptr, "null executor");
    *wire_in = ex->wire_in;
    *wire_out = ex->wire_out;
  });
}

rr_status rr_exec_enable_onload(rr_exec* ex, int n_src, const int32_t* src_devices, const int64_t* src_bytes,
                                 int64_t chunk_bytes) {
  return guarded([&] {
    need(ex != nullptr, "null executor");
    need(n_src >= 0 && chunk_bytes >= 4096, "bad onload arguments");
    check_cuda(cudaSetDevice(ex->cuda_device), "cudaSetDevice");
    for (auto e : ex->events) cudaEventDestroy(e);
    ex->events.clear();
    ex->chunks.clear();
    std::map<DeviceId, int> first_chunk;
    for (int i = 0; i < n_src; ++i) {
      need(src_devices[i] >= 0 && src_devices[i] < static_cast<int>(ex->src_bases.size()), "onload device range");
      need(ex->src_bases[static_cast<size_t>(src_devices[i])] != nullptr, "onload device has no source buffer");
      first_chunk[src_devices[i]] = static_cast<int>(ex->chunks.size());
      for (int64_t off = 0; off < src_bytes[i]; off += chunk_bytes)
        ex->chunks.push_back({src_devices[i], off, std::min(chunk_bytes, src_bytes[i] - off)});
    }
    // A copy-engine run over an onloaded source must lie inside the onloaded
    // bytes, like every item (checked below).
    for (const auto& c : ex->ce)
      for (int k = 0; k < n_src; ++k)
        if (src_devices[k] == c.src_dev)
          need(c.src_end <= src_bytes[k], "a copy-engine copy reads beyond the onloaded bytes of its source");
    // So must every staged push: it sends source bytes as they stand.
    for (const auto& p : ex->stage)
      for (int k = 0; k < n_src; ++k)
        if (src_devices[k] == p.src_dev)
          need(p.src_off + static_cast<int64_t>(p.bytes) <= src_bytes[k],
               "a staged push reads beyond the onloaded bytes of its source");
    // Segment of each item: 0 = independent of the onload, 1 + c = needs chunk c.
    const rr::ItemSet& a = ex->phase0_host;
    const size_t n = a.items.size(), C = ex->chunks.size();
    std::vector<std::vector<int>> seg_vec(C + 2), seg_other(C + 2);
    for (size_t i = 0; i < n; ++i) {
      int seg = 0;
      const auto it = first_chunk.find(a.src_dev[i]);
      if (a.items[i].wait_flag && ex->stage_ctas > 0) {
        // Staged unpack: its pieces come from the other GPUs' copy engines,
        // which never wait for a kernel here, so it runs from the start on
        // its own stream (rr_exec_launch_onload), unpacking while the onload
        // is still running.
        seg = static_cast<int>(C) + 1;
      } else if (a.items[i].wait_flag) {
        // Relay / overlapped fan-out items wait on other GPUs' pushes, which
        // may depend on this GPU's own pushes: launch them after every chunk
        // (and so every push of this GPU) so no launch waits on a later one.
        seg = static_cast<int>(C);
      } else if (it != first_chunk.end() && !a.src_is_dst[i]) {
        const DeviceId d = a.src_dev[i];
        int64_t total = 0;
        for (int k = 0; k < n_src; ++k)
          if (src_devices[k] == d) total = src_bytes[k];
        need(a.src_end[i] <= total, "an item reads beyond the onloaded bytes of its source");
        seg = 1 + it->second + static_cast<int>((a.src_end[i] - 1) / chunk_bytes);
      }
      (static_cast<int>(i) < a.n_vec ? seg_vec : seg_other)[static_cast<size_t>(seg)].push_back(static_cast<int>(i));
    }
    std::vector<rr::CopyItem> ordered;
    ordered.reserve(n);
    ex->segments.assign(C + 2, {});
    for (size_t s = 0; s <= C + 1; ++s) {
      auto& sg = ex->segments[s];
      sg.offset = static_cast<int>(ordered.size());
      for (int i : seg_vec[s]) ordered.push_back(a.items[static_cast<size_t>(i)]);
      sg.n_vec = static_cast<int>(seg_vec[s].size());
      for (int i : seg_other[s]) ordered.push_back(a.items[static_cast<size_t>(i)]);
      sg.n = static_cast<int>(ordered.size()) - sg.offset;
    }
    if (ex->d_onload) cudaFree(ex->d_onload);
    ex->d_onload = nullptr;
    if (!ordered.empty()) {
      check_cuda(cudaMalloc(&ex->d_onload, ordered.size() * sizeof(rr::CopyItem)), "cudaMalloc(onload items)");
      check_cuda(cudaMemcpy(ex->d_onload, ordered.data(), ordered.size() * sizeof(rr::CopyItem),
                            cudaMemcpyHostToDevice),
                 "upload onload items");
    }
    ex->events.resize(C);
    for (auto& e : ex->events) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  });
}

rr_status rr_exec_launch_onload(rr_exec* ex, void* const* host_bufs, void* copy_stream, void* stream, int ctas) {
  return guarded([&] {
    need(ex != nullptr && host_bufs != nullptr, "null executor/host buffers");
    need(!ex->segments.empty(), "rr_exec_enable_onload has not been called");
    check_cuda(cudaSetDevice(ex->cuda_device), "cudaSetDevice");
    ++ex->epoch;  // a phase-0 launch like rr_exec_launch
    auto cs = static_cast<cudaStream_t>(copy_stream);
    auto ks = static_cast<cudaStream_t>(stream);
    // The copy stream must not overwrite sources still read by an earlier
    // launch on the compute stream.
    cudaEvent_t ready;
    check_cuda(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "cudaEventCreate");
    check_cuda(cudaEventRecord(ready, ks), "cudaEventRecord");
    check_cuda(cudaStreamWaitEvent(cs, ready, 0), "cudaStreamWaitEvent");
    cudaEventDestroy(ready);
    for (size_t c = 0; c < ex->chunks.size(); ++c) {
      const auto& ch = ex->chunks[c];
      const void* h = host_bufs[ch.device];
      need(h != nullptr, "missing host buffer for an onloaded device");
      char* dst = static_cast<char*>(ex->src_bases[static_cast<size_t>(ch.device)]) + ch.offset;
      check_cuda(cudaMemcpyAsync(dst, static_cast<const char*>(h) + ch.offset, static_cast<size_t>(ch.bytes),
                                 cudaMemcpyHostToDevice, cs),
                 "onload cudaMemcpyAsync");
      check_cuda(cudaEventRecord(ex->events[c], cs), "cudaEventRecord");
    }
    if (!ex->ce.empty() || !ex->stage.empty()) {
      check_cuda(cudaEventRecord(ex->ce_fork, ks), "cudaEventRecord(ce fork)");
      check_cuda(cudaStreamWaitEvent(ex->ce_stream, ex->ce_fork, 0), "cudaStreamWaitEvent(ce fork)");
    }
    if (!ex->stage.empty()) {
      // Staged pushes follow the onload of the bytes they send: each waits
      // for the chunk holding its last byte (chunks land in order per
      // device). While the host link is the bottleneck the rotation order
      // would hold every later round back until the whole onload is done, so
      // pushes go out in the order their bytes land, each piece to every
      // receiver in turn.
      std::vector<std::pair<int, size_t>> order;  // (last chunk, push index)
      for (size_t i = 0; i < ex->stage.size(); ++i) {
        const auto& p = ex->stage[i];
        int last = -1;
        for (size_t k = 0; k < ex->chunks.size(); ++k) {
          const auto& ch = ex->chunks[k];
          if (ch.device == p.src_dev && ch.offset < p.src_off + static_cast<int64_t>(p.bytes)) last = static_cast<int>(k);
        }
        order.push_back({last, i});
      }
      std::stable_sort(order.begin(), order.end(),
                       [](const auto& a, const auto& b) { return a.first < b.first; });
      int waited = -1;
      for (const auto& [last, i] : order) {
        const auto& p = ex->stage[i];
        if (last > waited) {
          check_cuda(cudaStreamWaitEvent(ex->ce_stream, ex->events[static_cast<size_t>(last)], 0),
                     "cudaStreamWaitEvent(staged push)");
          waited = last;
        }
        // (round waits are skipped here: pushes follow the onload's chunk
        // order, not the rounds'; the tokens are still passed on)
        if (p.bytes) {
          check_cuda(cudaMemcpyAsync(p.dst, p.src, p.bytes, cudaMemcpyDeviceToDevice, ex->ce_stream), "staged push");
          signal_piece(ex->ce_stream, p.flag, ex->epoch);
        }
        if (p.done) signal_piece(ex->ce_stream, p.done, ex->epoch);
      }
    }
    if (!ex->ce.empty()) {
      // Copy-engine copies follow the onload: the part of a contiguous run
      // that reads chunk c starts once chunk c has landed; a 2D / 3D
      // transport copy starts once the chunk holding its last source byte
      // has; copies over sources that are not onloaded start right away.
      auto onloaded = [&](DeviceId d) {
        return std::any_of(ex->chunks.begin(), ex->chunks.end(), [&](const rr_exec::Chunk& ch) { return ch.device == d; });
      };
      auto flat = [](const rr_exec::CeCopy& c) { return c.height == 1 && c.depth == 1; };
      auto piece = [&](const rr_exec::CeCopy& c, int64_t lo, int64_t hi) {  // source bytes [lo, hi) of the shard
        const int64_t a = std::max(lo, c.src_off), b = std::min(hi, c.src_end);
        if (a >= b) return;
        rr_exec::CeCopy p = c;
        p.dst += a - c.src_off;
        p.src += a - c.src_off;
        p.width = b - a;
        issue_copy(p, ex->ce_stream);
      };
      // (schedule waits are skipped here: copies follow the onload's chunk
      // order, not the schedule's, so a wait could point ahead in this
      // stream; the done flags are still raised, no one waits on them.)
      // A star flag releases its whole group (the copies since the previous
      // flagged copy of the same stream list): it is written once the last
      // copy of the group to be issued here has been, whatever the order.
      std::vector<int> left(ex->ce.size(), 0);  // per flagged copy: its group's copies not yet fully issued
      std::vector<size_t> group_of(ex->ce.size(), 0);
      for (size_t i = ex->ce.size(); i-- > 0;) {
        if (ex->ce[i].flag) group_of[i] = i;
        else if (i + 1 < ex->ce.size()) group_of[i] = group_of[i + 1];
        else group_of[i] = i;
      }
      for (size_t i = 0; i < ex->ce.size(); ++i)
        if (ex->ce[group_of[i]].flag) ++left[group_of[i]];
      auto finished = [&](size_t i) {  // copy i fully issued on ce_stream
        const auto& c = ex->ce[i];
        if (c.done) signal_piece(ex->ce_stream, c.done, ex->epoch);
        const size_t g = group_of[i];
        if (ex->ce[g].flag && --left[g] == 0) signal_piece(ex->ce_stream, ex->ce[g].flag, ex->epoch);
      };
      // Relay forwards (hard waits: the piece must have arrived) go last, in
      // (op, piece) order: every send they wait for is issued before them
      // on its stream and waits only for local onload chunks.
      for (size_t i = 0; i < ex->ce.size(); ++i)
        if (!ex->ce[i].hard_wait && !onloaded(ex->ce[i].src_dev)) {
          issue_copy(ex->ce[i], ex->ce_stream);
          finished(i);
        }
      for (size_t k = 0; k < ex->chunks.size(); ++k) {
        const auto& ch = ex->chunks[k];
        const int64_t lo = ch.offset, hi = ch.offset + ch.bytes;
        auto in_chunk = [&](const rr_exec::CeCopy& c) {
          if (c.src_dev != ch.device) return false;
          return flat(c) ? (c.src_off < hi && c.src_end > lo) : (c.src_end > lo && c.src_end <= hi);
        };
        if (!std::any_of(ex->ce.begin(), ex->ce.end(), in_chunk)) continue;
        check_cuda(cudaStreamWaitEvent(ex->ce_stream, ex->events[k], 0), "cudaStreamWaitEvent(ce chunk)");
        for (size_t i = 0; i < ex->ce.size(); ++i) {
          const auto& c = ex->ce[i];
          if (c.hard_wait || !in_chunk(c)) continue;
          if (flat(c))
            piece(c, lo, hi);
          else
            issue_copy(c, ex->ce_stream);
          if (c.src_end > lo && c.src_end <= hi) finished(i);  // its last piece
        }
      }
      for (size_t i = 0; i < ex->ce.size(); ++i)
        if (ex->ce[i].hard_wait) {
          wait_piece(ex->ce_stream, ex->ce[i].wait, ex->epoch);
          issue_copy(ex->ce[i], ex->ce_stream);
          finished(i);
        }
    }
    auto segment_phase = [&](const rr_exec::Segment& sg) {
      rr_exec::Phase ph;
      ph.d = ex->d_onload + sg.offset;
      ph.n = sg.n;
      ph.n_vec = sg.n_vec;
      ph.flagged = ex->phase[0].flagged;
      // The kernel is chosen once for the whole phase (phase_kernel reads
      // `written`): a GiB-sized phase keeps the TMA ring in every segment.
      ph.written = ex->phase[0].written;
      return ph;
    };
    const auto& staged_seg = ex->segments.back();  // C + 1: staged unpack
    if (staged_seg.n > 0) {
      check_cuda(cudaEventRecord(ex->unpack_fork, ks), "cudaEventRecord(unpack fork)");
      check_cuda(cudaStreamWaitEvent(ex->unpack_stream, ex->unpack_fork, 0), "cudaStreamWaitEvent(unpack fork)");
      launch_phase(ex, segment_phase(staged_seg), ex->unpack_stream, ctas, ex->d_sched2);
    }
    for (size_t s = 0; s + 1 < ex->segments.size(); ++s) {
      if (s > 0) check_cuda(cudaStreamWaitEvent(ks, ex->events[s - 1], 0), "cudaStreamWaitEvent");
      const auto& sg = ex->segments[s];
      if (sg.n == 0) continue;
      rr_exec::Phase ph = segment_phase(sg);
      if (ex->stage_ctas > 0) ph.flagged = false;  // local copies only: the plain-phase kernel
      launch_phase(ex, ph, stream, ctas);
    }
    if (staged_seg.n > 0) {
      check_cuda(cudaEventRecord(ex->unpack_join, ex->unpack_stream), "cudaEventRecord(unpack join)");
      check_cuda(cudaStreamWaitEvent(ks, ex->unpack_join, 0), "cudaStreamWaitEvent(unpack join)");
    }
    if (!ex->ce.empty() || !ex->stage.empty()) ce_join(ex, ks);
  });
}

rr_status rr_exec_launch_offload(rr_exec* ex, int n_src, const int32_t* src_devices, const int64_t* src_bytes,
                                 void* const* host_bufs, void* copy_stream, void* stream) {
  return guarded([&] {
    need(ex != nullptr && host_bufs != nullptr, "null executor/host buffers");
    need(n_src >= 0 && (n_src == 0 || (src_devices != nullptr && src_bytes != nullptr)), "bad offload arguments");
    check_cuda(cudaSetDevice(ex->cuda_device), "cudaSetDevice");
    for (int i = 0; i < n_src; ++i) {
      need(src_devices[i] >= 0 && src_devices[i] < static_cast<int>(ex->src_bases.size()), "offload device range");
      need(ex->src_bases[static_cast<size_t>(src_devices[i])] != nullptr, "offload device has no source buffer");
      need(host_bufs[src_devices[i]] != nullptr, "missing host buffer for an offloaded device");
      need(src_bytes[i] >= 0, "negative offload size");
    }
    // Sources are complete once the work already on `stream` is; from then
    // on the copy engine and a reallocation launched next on `stream` only
    // read them, so the two overlap.
    auto cs = static_cast<cudaStream_t>(copy_stream);
    cudaEvent_t ready;
    check_cuda(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "cudaEventCreate");
    check_cuda(cudaEventRecord(ready, static_cast<cudaStream_t>(stream)), "cudaEventRecord");
    check_cuda(cudaStreamWaitEvent(cs, ready, 0), "cudaStreamWaitEvent");
    cudaEventDestroy(ready);
    for (int i = 0; i < n_src; ++i) {
      if (src_bytes[i] == 0) continue;
      const DeviceId d = src_devices[i];
      check_cuda(cudaMemcpyAsync(host_bufs[d], ex->src_bases[static_cast<size_t>(d)], static_cast<size_t>(src_bytes[i]),
                                 cudaMemcpyDeviceToHost, cs),
                 "offload cudaMemcpyAsync");
    }
  });
}

void rr_exec_destroy(rr_exec* ex) { delete ex; }
