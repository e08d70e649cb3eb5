// Host-side construction of executor work: which device reads what and
// stores where, in which phase, for one executing host. Shared by
// rr_exec_create (real pointers, device items) and rr_plan_work (byte
// accounting only, no CUDA).
#pragma once

#include <cstdint>
#include <functional>
#include <set>
#include <tuple>
#include <vector>

#include "rlplan/realloc.hpp"
#include "rr_internal.hpp"

namespace rr {

// Phase A: every copy that reads a real source shard. A destination host
// with several plan devices of one op receives the payload once, into its
// lowest-id device (the leader); a host that holds the source writes all of
// its own destinations directly.
// Phase B (after a cross-host barrier): the host copies leader regions into
// the other local destinations of that op — one NVLink crossing per host
// instead of one per destination device (hierarchical broadcast).
struct Job {
  int phase = 0;
  rlplan::DeviceId src = -1;       // device whose buffer is read
  bool src_is_dst_buffer = false;  // phase B: the leader's destination shard
  std::vector<rlplan::DeviceId> dsts;
  const rlplan::LoweredOp* op = nullptr;
  // dsts[0] stands for every member of an NVLS multicast group: stored once
  // through mc_base (multimem.st), replicated by the switch.
  bool multicast = false;
  uint64_t mc_base = 0;
  // Pipelined relay: item k of this job is relay slot relay_base + k. With
  // relay_wait the job reads this host's leader copy only after the previous
  // host of the chain flagged that slot; with relay_signal dsts[0] is the
  // next host's leader, flagged after each item.
  bool relay_wait = false;
  bool relay_signal = false;
  int64_t relay_base = 0;
  // Copy-engine star: an in-host fan-out in phase 0 whose items wait for the
  // transport copy that filled the leader bytes they read.
  bool ce_wait = false;
  // ... of a copy-engine relay payload: the items wait for the relay piece
  // holding the last leader byte they read.
  bool ce_relay = false;
};

struct HostMap {
  std::vector<int> host;     // host id per plan device
  int me = 0;                // executing host
  bool hierarchical = true;  // false: flat delivery, every destination served directly
  std::vector<uint64_t> mc;  // per plan device: multicast address of its group (0 = none)
  // Per plan device, the (locally mapped) relay flag array of its host;
  // empty = no flag-synchronised schemes.
  std::vector<uint64_t> relay_flags;
  int64_t relay_chunk = 256 << 10;
  // chain: payloads reaching >= 2 other hosts travel source -> host -> host.
  // star: a payload's in-host fan-out starts per chunk as soon as the chunk
  // lands, inside phase 0 (no separate fan-out phase).
  bool relay_chain = true;
  bool relay_star = false;
  // Staged gather (pull mode): the remote source shards this host reads
  // arrive whole in local staging buffers (passed as their source buffers),
  // pushed by their hosts' copy engines in stage_chunk pieces, each piece
  // flagged in this host's stage flag array (stage_flags, mapped here).
  // Every local destination is written directly (no fan-out phase), and an
  // item reading staged bytes waits for the piece holding its last byte.
  int64_t stage_chunk = 0;               // 0 = off
  uint64_t stage_flags = 0;
  std::vector<int64_t> stage_slot0;      // per plan device: its first slot here, -1 = not staged
  // Copy-engine transport (push): every remote destination of a plain
  // phase-0 job is left out of the SM items; ce_transport_copies moves it.
  bool ce_remote = false;
  // Hybrid: row-parallel pieces whose layers do not merge into one 3D copy
  // (per-layer 2D copies run at ~686 GB/s against ~775) stay on SM peer
  // stores beside the copy engines; ce_sm_rects lists them as (source,
  // destination, destination offset of the rect).
  bool ce_hybrid = false;
  std::set<std::tuple<rlplan::DeviceId, rlplan::DeviceId, int64_t>> ce_sm_rects;
  // ... with per-copy flags (copy-engine star): each transport copy is
  // flagged in the receiving host's array (ce_flag_slot), and a host's
  // in-host fan-out runs inside phase 0, each item waiting for the copy that
  // filled the leader bytes it reads. ce_flags = this host's array.
  bool ce_star = false;
  uint64_t ce_flags = 0;
  // Copy-engine relay (with ce_remote): a payload reaching >= 2 other hosts
  // travels source -> host 1 -> host 2 ... (ring order) by copy engines,
  // piece by piece, each hop's copy stream waiting for the piece's flag
  // before forwarding it; every host fans its pieces out inside phase 0.
  bool ce_relay = false;
};

// Staged gather: the remote sources host `h` reads, in arrival order. Round
// r = 1..H-1 (H = number of hosts, hosts ranked by id) brings the sources
// held by the host r places before h, so in every round each host receives
// from exactly one host and sends to exactly one.
std::vector<rlplan::DeviceId> stage_sources(const std::vector<rlplan::LoweredOp>& ops, const std::vector<int>& host,
                                            int h);
// Slot of every staged source's first piece in host h's flag array (-1 for
// the others), and the array length.
std::vector<int64_t> stage_slots(const std::vector<rlplan::LoweredOp>& ops, const std::vector<int>& host, int h,
                                 const std::vector<int64_t>& src_bytes, int64_t chunk, int64_t* n_slots);

// Relay slots a plan needs (flag array length, identical on every rank).
int64_t relay_slots(const std::vector<rlplan::LoweredOp>& ops, const HostMap& hm);

// mode 0 = push (source host executes phase A), 1 = pull (destination host).
std::vector<Job> build_jobs(const std::vector<rlplan::LoweredOp>& ops, const HostMap& hm, int mode);

// Bytes that cross from/to host `me` (each payload crosses once per
// destination host).
void host_wire_bytes(const std::vector<rlplan::LoweredOp>& ops, const HostMap& hm, int64_t* in, int64_t* out);

int64_t rect_bytes(const rlplan::CopyRect& r);

// A contiguous byte range moved whole by a copy engine from a source shard
// (src device, source placement) into a destination shard (dst device,
// destination placement): both layouts hold the same blocks there at the
// same relative offsets, so byte x of the source range is byte x of the
// destination range. It replaces the SM items of every rect whose
// destination extent it contains, for that destination.
struct CeRun {
  rlplan::DeviceId src = -1, dst = -1;
  int64_t src_off = 0, dst_off = 0, bytes = 0;
};

// Maximal runs (>= min_bytes) between source layout `s` and destination
// layout `d` whose blocks match one to one (same tensor rectangle, same
// offset relative to the run start).
std::vector<CeRun> matching_runs(const rlplan::ShardLayout& s, const rlplan::ShardLayout& d, rlplan::DeviceId sd,
                                 rlplan::DeviceId dd, int64_t min_bytes);

// Copy-engine transport: one copy-engine submission of a (local source,
// remote destination) pair — width bytes x height rows x depth slices, rows
// at the pitches, slices at the slice strides (multiples of the pitches).
// depth > 1 is a cudaMemcpy3DAsync, height > 1 a cudaMemcpy2DAsync.
struct CeCopy {
  rlplan::DeviceId src = -1, dst = -1;
  int64_t src_off = 0, dst_off = 0;
  int64_t width = 0, height = 1, depth = 1;
  int64_t src_pitch = 0, dst_pitch = 0;
  int64_t src_slice = 0, dst_slice = 0;
  bool strided = false;  // rows are the rows of one row-parallel rect (not layers)
  int64_t bytes() const { return width * height * depth; }
  int64_t src_end() const { return src_off + (depth - 1) * src_slice + (height - 1) * src_pitch + width; }
};

// The copies that move every remote destination of the plain phase-0 push
// jobs in `jobs` (hm.ce_remote). The per-layer rects of one tensor kind sit
// at a constant layer stride in both shards, so they merge into one 2D copy
// (contiguous pieces: rows = layers) or one 3D copy (row-parallel pieces,
// when the layer strides are whole multiples of the row pitches); pitches
// stay <= max_pitch. Ordered in rotation rounds: round r sends to the host r
// places after this one (ids ascending), so while every host follows its
// order each receives from one sender at a time.
// With hm.ce_hybrid the unmerged row-parallel pieces are left out and, when
// sm_rects is given, recorded there.
std::vector<CeCopy> ce_transport_copies(const std::vector<Job>& jobs, const HostMap& hm, int64_t max_pitch,
                                        std::set<std::tuple<rlplan::DeviceId, rlplan::DeviceId, int64_t>>* sm_rects =
                                            nullptr);

// Copy-engine star slots: host h's flag array holds one slot per transport
// copy it receives, senders in ascending host order, each sender's copies to
// h in its issue order. ce_copies_of(ops, hm, g) = the copies host g issues.
std::vector<CeCopy> ce_copies_of(const std::vector<rlplan::LoweredOp>& ops, const HostMap& hm, int g,
                                 int64_t max_pitch);
// Slots of host h's array (the incoming copies).
int64_t ce_star_slots(const std::vector<rlplan::LoweredOp>& ops, const HostMap& hm, int h, int64_t max_pitch);
// Slot (in host `h`'s array) of the copy that carries byte `dst_off` of
// destination `dst` from source `src`, or -1.
struct CeSlotMap {
  std::vector<std::pair<CeCopy, int64_t>> copies;  // incoming copies of h with the slot their items wait on
  std::vector<double> ready;  // per slot: simulated landing time (ce_schedule), to order the waiting items
  int64_t slot_of(rlplan::DeviceId src, rlplan::DeviceId dst, int64_t dst_off) const;
};
// Copy-engine star flag groups: of a sender's copies (issue order), the
// ones followed by a flag write — the last of every >= kStarFlagBytes run and
// the last copy to each receiver. A flag write carries a system-wide memory
// barrier, so flagging every copy would drain the engine each time; the
// items of a copy wait for the flag of its group. Both sides derive the
// groups from the same copy list.
constexpr int64_t kStarFlagBytes = int64_t{256} << 20;
std::vector<bool> star_flagged(const std::vector<CeCopy>& copies, const HostMap& hm);
CeSlotMap ce_slot_map(const std::vector<rlplan::LoweredOp>& ops, const HostMap& hm, int h, int64_t max_pitch);
// Slot of each of this host's outgoing copies (in the receiving host's array).
std::vector<int64_t> ce_send_slots(const std::vector<rlplan::LoweredOp>& ops, const HostMap& hm,
                                   const std::vector<CeCopy>& mine, int64_t max_pitch);

// Copy-engine schedule. Every host's transport copies form transfers (one
// per receiving host); a global list schedule (each transfer starts when
// both its sender and its receiver are free, at the measured rates) orders
// them so that no receiver takes two senders at once — with rotation rounds
// alone, a sender whose round is empty runs ahead into a busy receiver (70B
// at 4 GPUs: 524 vs 745 GB/s). Each transfer waits (cuStreamWaitValue32 on
// its sender's array) for the previous transfer into the same receiver when
// that one has another sender, which raises the flag after its last copy.
// Waits only point to transfers that start earlier: no cycles.
struct CeTransfer {
  int sender = 0, receiver = 0;
  size_t first = 0, count = 0;  // copies [first, first + count) of the sender's ce_transport_copies list
  double start = 0, end = 0;    // simulated seconds
  int64_t wait_slot = -1;       // in the sender's flag array (-1 = no wait)
  int signal_host = -1;         // after the last copy: raise signal_slot in this host's array
  int64_t signal_slot = -1;
};
// All hosts' transfers, each host's in issue order (ascending start). The
// schedule's slots of host h follow its ce_star_slots incoming-copy slots.
std::vector<CeTransfer> ce_schedule(const std::vector<rlplan::LoweredOp>& ops, const HostMap& hm,
                                    int64_t max_pitch);
// Length of host h's copy flag array: incoming copy slots + schedule waits
// (+ relay piece slots with hm.ce_relay).
int64_t ce_flag_slots(const std::vector<rlplan::LoweredOp>& ops, const HostMap& hm, int h, int64_t max_pitch);

// Copy-engine relay. A piece is a 1D run (height 1) or a row range of a
// row-parallel rect, <= kRelayPieceBytes, in the op's rect order; hop 0
// reads the source shard (src geometry), later hops read the previous
// host's leader (the destination geometry on both sides). Pieces of one op
// land in order on every hop.
constexpr int64_t kRelayPieceBytes = int64_t{256} << 20;
bool ce_relay_op(const rlplan::LoweredOp& op, const HostMap& hm);
struct CeRelayPiece {
  int64_t src_off = 0, dst_off = 0, width = 0, height = 1, src_pitch = 0, dst_pitch = 0;
  int64_t dst_last() const { return dst_off + (height - 1) * dst_pitch + width - 1; }
};
struct CeRelayOp {
  const rlplan::LoweredOp* op = nullptr;
  int src_host = 0;
  std::vector<int> chain;                   // destination hosts in hop order
  std::vector<rlplan::DeviceId> leader;     // per chain host: its lowest-id destination
  std::vector<CeRelayPiece> pieces;
  int64_t slot0 = 0;                        // relay slot of piece 0 (same on every host)
};
// The relay ops of a plan (plan order) with their pieces and slots.
std::vector<CeRelayOp> ce_relay_ops(const std::vector<rlplan::LoweredOp>& ops, const HostMap& hm);
// First relay slot in host h's flag array (after its star and schedule slots).
int64_t ce_relay_base(const std::vector<rlplan::LoweredOp>& ops, const HostMap& hm, int h, int64_t max_pitch);

// Byte extent [first, last) a rect writes in its destination shard.
inline int64_t rect_dst_end(const rlplan::CopyRect& r) {
  return r.dst_off + (r.rows - 1) * r.dst_pitch + r.row_bytes;
}

// Items of one phase, chunked and interleaved across jobs; 16-byte items
// first, then 2-byte items. `ce` (may be null): runs whose (rect,
// destination) pairs are left out of the items.
struct ItemSet {
  std::vector<CopyItem> items;
  int n_vec = 0;
  int64_t read = 0, written = 0;
  bool remote_stores = false;  // some destination is on another host
  // Per item (same order): the device whose buffer it reads and one past the
  // last source byte it reads (onload pipelining, rr_exec_enable_onload).
  std::vector<rlplan::DeviceId> src_dev;
  std::vector<int64_t> src_end;
  std::vector<bool> src_is_dst;  // reads a destination (leader) buffer
};

// Resolve jobs of `phase` into items. src_bufs/dst_bufs are indexed by plan
// device; nullptr tables mean "accounting only" (addresses left at offsets).
// relay: (op, destination byte) -> relay slot in this host's array (-1: none);
// items of ce_relay jobs wait on base + 4 * slot of their last byte.
using RelaySlotFn = std::function<int64_t(const rlplan::LoweredOp*, int64_t)>;
ItemSet build_items(const std::vector<Job>& jobs, int phase, const HostMap& hm, void* const* src_bufs,
                    void* const* dst_bufs, int64_t chunk_bytes, const std::vector<CeRun>* ce = nullptr,
                    const CeSlotMap* ce_slots = nullptr, const RelaySlotFn* relay_piece_slot = nullptr);

}  // namespace rr
