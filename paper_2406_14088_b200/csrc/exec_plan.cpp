// Executor work construction (see exec_plan.hpp). The upstream runtime
// broadcasts each TP partition from its chosen source to every destination
// (PAPER.md:515); here a payload crosses NVLink once per destination host
// and is replicated inside the host from HBM.
#include "exec_plan.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <tuple>

namespace rr {

using rlplan::CopyRect;
using rlplan::DeviceId;
using rlplan::LoweredOp;

int64_t rect_bytes(const CopyRect& r) { return r.row_bytes * r.rows; }

namespace {

int64_t op_bytes(const LoweredOp& op) {
  int64_t b = 0;
  for (const auto& r : op.rects) b += rect_bytes(r);
  return b;
}

std::map<int, std::vector<DeviceId>> by_host(const LoweredOp& op, const HostMap& hm) {
  std::map<int, std::vector<DeviceId>> g;
  for (DeviceId d : op.dst) g[hm.host[static_cast<size_t>(d)]].push_back(d);
  for (auto& kv : g) std::sort(kv.second.begin(), kv.second.end());
  return g;
}

// An op can be multicast when the leaders of its destination hosts are
// exactly the members of one multicast group (the switch writes every
// member, so a strict subset would clobber a non-destination).
bool multicast_target(const std::map<int, std::vector<DeviceId>>& groups, const HostMap& hm, uint64_t* base) {
  if (hm.mc.empty() || !hm.hierarchical) return false;
  uint64_t v = 0;
  for (const auto& kv : groups) {
    const uint64_t m = hm.mc[static_cast<size_t>(kv.second.front())];
    if (m == 0 || (v != 0 && m != v)) return false;
    v = m;
  }
  const size_t members = static_cast<size_t>(std::count(hm.mc.begin(), hm.mc.end(), v));
  if (members != groups.size()) return false;
  *base = v;
  return true;
}

// Pieces add_rect cuts a 16-byte-unit rectangle into (the same rule).
int64_t pieces_of(const CopyRect& r, int64_t chunk) {
  const int64_t cap_units = std::min<int64_t>(chunk / 16, kMaxItemUnits);
  const int64_t row_units = r.row_bytes / 16;
  if (row_units <= cap_units) {
    const int64_t rows_per = std::max<int64_t>(1, cap_units / std::max<int64_t>(row_units, 1));
    return (r.rows + rows_per - 1) / rows_per;
  }
  return r.rows * ((row_units + cap_units - 1) / cap_units);
}

// Remote destination hosts in ring order after the source host.
std::vector<int> relay_chain(const std::map<int, std::vector<DeviceId>>& groups, int hs) {
  std::vector<int> chain;
  int span = 1;
  for (const auto& kv : groups) span = std::max(span, std::abs(kv.first - hs) + 1);
  for (const auto& kv : groups)
    if (kv.first != hs) chain.push_back(kv.first);
  std::sort(chain.begin(), chain.end(), [&](int a, int b) {
    return ((a - hs) % span + span) % span < ((b - hs) % span + span) % span;
  });
  return chain;
}

// Relay pays off when a payload reaches >= 2 other hosts (it caps every
// host's egress at one copy). Needs 16-byte geometry on both sides (the
// source and the forwarders cut identical pieces) and small fan-outs.
bool flaggable(const LoweredOp& op, const std::map<int, std::vector<DeviceId>>& groups, const HostMap& hm) {
  if (!hm.hierarchical) return false;
  uint64_t mc = 0;
  if (multicast_target(groups, hm, &mc)) return false;
  for (const auto& kv : groups)
    if (static_cast<int>(kv.second.size()) + 1 > kMaxFan) return false;
  for (const auto& r : op.rects)
    if (((r.src_off | r.dst_off | r.row_bytes | r.src_pitch | r.dst_pitch) & 15) != 0) return false;
  return true;
}

bool relay_eligible(const LoweredOp& op, const std::map<int, std::vector<DeviceId>>& groups, const HostMap& hm) {
  if (!hm.relay_chain || !flaggable(op, groups, hm)) return false;
  const int hs = hm.host[static_cast<size_t>(op.src)];
  int remote = 0;
  for (const auto& kv : groups)
    if (kv.first != hs) ++remote;
  return remote >= 2;
}

// Remote hosts whose in-host fan-out overlaps phase 0 (star scheme): they
// hold >= 2 destinations of a payload that does not take the chain relay.
std::vector<int> star_hosts(const LoweredOp& op, const std::map<int, std::vector<DeviceId>>& groups,
                            const HostMap& hm) {
  std::vector<int> hosts;
  if (!hm.relay_star || relay_eligible(op, groups, hm) || !flaggable(op, groups, hm)) return hosts;
  const int hs = hm.host[static_cast<size_t>(op.src)];
  for (const auto& kv : groups)
    if (kv.first != hs && kv.second.size() >= 2) hosts.push_back(kv.first);
  return hosts;
}

int64_t op_pieces(const LoweredOp& op, int64_t chunk) {
  int64_t n = 0;
  for (const auto& r : op.rects) n += pieces_of(r, chunk);
  return n;
}

}  // namespace

int64_t relay_slots(const std::vector<LoweredOp>& ops, const HostMap& hm) {
  int64_t n = 0;
  for (const auto& op : ops) {
    const auto groups = by_host(op, hm);
    if (relay_eligible(op, groups, hm))
      n += op_pieces(op, hm.relay_chunk);
    else
      n += op_pieces(op, hm.relay_chunk) * static_cast<int64_t>(star_hosts(op, groups, hm).size());
  }
  return n;
}

std::vector<DeviceId> stage_sources(const std::vector<LoweredOp>& ops, const std::vector<int>& host, int h) {
  std::vector<int> hosts(host.begin(), host.end());
  std::sort(hosts.begin(), hosts.end());
  hosts.erase(std::unique(hosts.begin(), hosts.end()), hosts.end());
  const int H = static_cast<int>(hosts.size());
  const int pos = static_cast<int>(std::find(hosts.begin(), hosts.end(), h) - hosts.begin());
  std::vector<bool> needed(host.size(), false);
  for (const auto& op : ops)
    if (host[static_cast<size_t>(op.src)] != h)
      for (DeviceId d : op.dst)
        if (host[static_cast<size_t>(d)] == h) needed[static_cast<size_t>(op.src)] = true;
  std::vector<DeviceId> out;
  for (int r = 1; r < H; ++r) {
    const int g = hosts[static_cast<size_t>((pos - r + H) % H)];
    for (size_t s = 0; s < host.size(); ++s)
      if (needed[s] && host[s] == g) out.push_back(static_cast<DeviceId>(s));
  }
  return out;
}

std::vector<int64_t> stage_slots(const std::vector<LoweredOp>& ops, const std::vector<int>& host, int h,
                                 const std::vector<int64_t>& src_bytes, int64_t chunk, int64_t* n_slots) {
  std::vector<int64_t> slot0(host.size(), -1);
  int64_t n = 0;
  for (DeviceId s : stage_sources(ops, host, h)) {
    slot0[static_cast<size_t>(s)] = n;
    n += (src_bytes[static_cast<size_t>(s)] + chunk - 1) / chunk;
  }
  *n_slots = n;
  return slot0;
}

std::vector<Job> build_jobs(const std::vector<LoweredOp>& ops, const HostMap& hm, int mode) {
  std::vector<Job> jobs;
  if (!hm.hierarchical) {
    // Flat delivery: the executing side serves every destination directly
    // (push: all of a local source's destinations; pull: the local ones).
    for (const auto& op : ops) {
      Job j;
      j.src = op.src;
      j.op = &op;
      for (DeviceId d : op.dst)
        if (mode == 0 ? hm.host[static_cast<size_t>(op.src)] == hm.me : hm.host[static_cast<size_t>(d)] == hm.me)
          j.dsts.push_back(d);
      if (!j.dsts.empty()) jobs.push_back(std::move(j));
    }
    return jobs;
  }
  int64_t relay_next_slot = 0;  // slots are numbered identically on every rank
  for (const auto& op : ops) {
    const int hs = hm.host[static_cast<size_t>(op.src)];
    const auto groups = by_host(op, hm);
    const auto mine = groups.find(hm.me);
    if (mode == 0 && !hm.relay_flags.empty() && relay_eligible(op, groups, hm)) {
      // Pipelined relay: source -> c1 -> c2 -> ... (ring order); each host
      // forwards every chunk as soon as it lands and fans it out locally in
      // the same pass, so no host sends more than one copy.
      const int64_t base = relay_next_slot;
      for (const auto& r : op.rects) relay_next_slot += pieces_of(r, hm.relay_chunk);
      const std::vector<int> chain = relay_chain(groups, hs);
      auto leader = [&](int h) { return groups.at(h).front(); };
      if (hs == hm.me) {
        Job j;
        j.src = op.src;
        j.op = &op;
        j.dsts.push_back(leader(chain.front()));
        if (mine != groups.end()) j.dsts.insert(j.dsts.end(), mine->second.begin(), mine->second.end());
        j.relay_signal = true;
        j.relay_base = base;
        jobs.push_back(std::move(j));
      } else if (mine != groups.end()) {
        const size_t pos = static_cast<size_t>(std::find(chain.begin(), chain.end(), hm.me) - chain.begin());
        Job j;
        j.src = mine->second.front();
        j.src_is_dst_buffer = true;
        j.op = &op;
        if (pos + 1 < chain.size()) {
          j.dsts.push_back(leader(chain[pos + 1]));
          j.relay_signal = true;
        }
        j.dsts.insert(j.dsts.end(), mine->second.begin() + 1, mine->second.end());
        j.relay_wait = true;
        j.relay_base = base;
        if (!j.dsts.empty()) jobs.push_back(std::move(j));
      }
      continue;
    }
    const std::vector<int> stars = star_hosts(op, groups, hm);
    if (mode == 0 && !hm.relay_flags.empty() && !stars.empty()) {
      // Star: the source pushes each chunk to every remote leader and flags
      // the hosts that fan out; those fan each chunk out as soon as it lands,
      // inside phase 0.
      const int64_t pieces = op_pieces(op, hm.relay_chunk);
      std::map<int, int64_t> base;
      for (int h : stars) {
        base[h] = relay_next_slot;
        relay_next_slot += pieces;
      }
      if (hs == hm.me) {
        Job plain;  // local destinations and single-destination remote hosts
        plain.src = op.src;
        plain.op = &op;
        for (const auto& [h, list] : groups) {
          if (h == hm.me)
            plain.dsts.insert(plain.dsts.end(), list.begin(), list.end());
          else if (!base.count(h))
            plain.dsts.push_back(list.front());
        }
        if (!plain.dsts.empty()) jobs.push_back(std::move(plain));
        for (int h : stars) {
          Job j;
          j.src = op.src;
          j.op = &op;
          j.dsts = {groups.at(h).front()};
          j.relay_signal = true;
          j.relay_base = base[h];
          jobs.push_back(std::move(j));
        }
      } else if (base.count(hm.me)) {
        Job j;
        j.src = mine->second.front();
        j.src_is_dst_buffer = true;
        j.op = &op;
        j.dsts.assign(mine->second.begin() + 1, mine->second.end());
        j.relay_wait = true;
        j.relay_base = base[hm.me];
        jobs.push_back(std::move(j));
      }
      continue;
    }
    uint64_t mc_base = 0;
    if (mode == 0 && hs == hm.me && multicast_target(groups, hm, &mc_base)) {
      // One multimem store reaches every host's leader (our own included);
      // our other local destinations are stored directly from the same read.
      Job j;
      j.phase = 0;
      j.src = op.src;
      j.op = &op;
      j.multicast = true;
      j.mc_base = mc_base;
      j.dsts.push_back(groups.begin()->second.front());
      if (mine != groups.end()) j.dsts.insert(j.dsts.end(), mine->second.begin() + 1, mine->second.end());
      jobs.push_back(std::move(j));
    } else if (mode == 0) {  // push: the source host drives phase A
      if (hs == hm.me) {
        // One job: the source is read once for every local destination and
        // every remote host's leader (build_items splits > kMaxFan targets).
        // A copy-engine relay payload reaches the remote hosts by the relay
        // (ce_relay_ops), not from here.
        Job j;
        j.phase = 0;
        j.src = op.src;
        j.op = &op;
        if (mine != groups.end()) j.dsts = mine->second;
        if (!ce_relay_op(op, hm))
          for (const auto& [h, list] : groups)
            if (h != hm.me) j.dsts.push_back(list.front());
        if (!j.dsts.empty()) jobs.push_back(std::move(j));
      }
    } else if (mine != groups.end()) {  // pull: each destination host fetches for itself
      Job j;
      j.phase = 0;
      j.src = op.src;
      j.op = &op;
      const bool all_local = hs == hm.me || hm.stage_chunk > 0;  // staged: the source is local memory
      j.dsts = all_local ? mine->second : std::vector<DeviceId>{mine->second.front()};
      jobs.push_back(std::move(j));
    }
    if (hs != hm.me && mine != groups.end() && mine->second.size() > 1 && !(mode == 1 && hm.stage_chunk > 0)) {
      Job j;
      // copy-engine star / relay: the fan-out waits per copy / piece inside phase 0
      const bool relayed = mode == 0 && ce_relay_op(op, hm);
      j.phase = (hm.ce_star || relayed) && mode == 0 ? 0 : 1;
      j.ce_wait = j.phase == 0;
      j.ce_relay = relayed;
      j.src = mine->second.front();
      j.src_is_dst_buffer = true;
      j.op = &op;
      j.dsts.assign(mine->second.begin() + 1, mine->second.end());
      jobs.push_back(std::move(j));
    }
  }
  return jobs;
}

void host_wire_bytes(const std::vector<LoweredOp>& ops, const HostMap& hm, int64_t* in, int64_t* out) {
  int64_t i = 0, o = 0;
  for (const auto& op : ops) {
    const int hs = hm.host[static_cast<size_t>(op.src)];
    const int64_t b = op_bytes(op);
    const auto groups = by_host(op, hm);
    if ((!hm.relay_flags.empty() && relay_eligible(op, groups, hm)) || ce_relay_op(op, hm)) {
      // relay (SM or copy-engine): every chain host receives one copy; all
      // but the last send one
      const std::vector<int> chain = relay_chain(groups, hs);
      if (hs == hm.me) o += b;
      const auto at = std::find(chain.begin(), chain.end(), hm.me);
      if (at != chain.end()) {
        i += b;
        if (at + 1 != chain.end()) o += b;
      }
      continue;
    }
    uint64_t mc_base = 0;
    const bool mc = multicast_target(groups, hm, &mc_base);
    bool sent = false;
    for (const auto& [h, list] : groups) {
      if (h == hs) continue;
      // hierarchical: once per destination host; flat: once per destination
      // device; multicast: leaves the source once, enters every host once
      const int64_t copies = hm.hierarchical ? 1 : static_cast<int64_t>(list.size());
      if (h == hm.me) i += b * copies;
      if (hs == hm.me && !(mc && sent)) o += b * copies;
      sent = true;
    }
  }
  *in = i;
  *out = o;
}

std::vector<CeRun> matching_runs(const rlplan::ShardLayout& s, const rlplan::ShardLayout& d, DeviceId sd,
                                 DeviceId dd, int64_t min_bytes) {
  using Key = std::tuple<int, rlplan::Count, rlplan::Count, rlplan::Count, rlplan::Count>;
  const auto key = [](const rlplan::TensorBlock& b) { return Key{b.tensor, b.r0, b.r1, b.c0, b.c1}; };
  const auto bytes = [](const rlplan::TensorBlock& b) { return (b.r1 - b.r0) * (b.c1 - b.c0) * 2; };  // bf16 (G10)
  std::map<Key, size_t> where;
  for (size_t k = 0; k < d.blocks.size(); ++k) where.emplace(key(d.blocks[k]), k);
  std::vector<CeRun> out;
  for (size_t i = 0; i < s.blocks.size();) {
    const auto it = where.find(key(s.blocks[i]));
    if (it == where.end()) {
      ++i;
      continue;
    }
    size_t j = it->second;
    const int64_t s0 = s.blocks[i].offset, d0 = d.blocks[j].offset;
    int64_t end = s0 + bytes(s.blocks[i]);
    for (++i, ++j; i < s.blocks.size() && j < d.blocks.size() && key(s.blocks[i]) == key(d.blocks[j]) &&
                   s.blocks[i].offset - s0 == d.blocks[j].offset - d0;
         ++i, ++j)
      end = s.blocks[i].offset + bytes(s.blocks[i]);
    if (end - s0 >= min_bytes) out.push_back({sd, dd, s0, d0, end - s0});
  }
  return out;
}

namespace {

// A job whose remote destinations the copy-engine transport (or a copy-engine
// run) may take: plain phase-0 work reading a real source shard.
bool plain_push(const Job& j, int phase) {
  return phase == 0 && !j.multicast && !j.src_is_dst_buffer && !j.relay_wait && !j.relay_signal;
}

bool ce_covered(const std::vector<CeRun>& runs, DeviceId src, DeviceId dst, const CopyRect& r) {
  for (const auto& u : runs)
    if (u.src == src && u.dst == dst && r.dst_off >= u.dst_off && rect_dst_end(r) <= u.dst_off + u.bytes) return true;
  return false;
}

// An item plus where it reads from (for onload pipelining).
struct Tagged {
  CopyItem it;
  DeviceId src_dev;
  int64_t src_end;
  bool src_is_dst;
};

// Chunk one rectangle for (src base, dst bases) into items.
// Relay flags of the items a rectangle is cut into: item k waits on
// wait_base + 4*slot and/or signals signal_base + 4*slot, slot = (*slot)++.
struct RelayTags {
  uint64_t wait_base = 0, signal_base = 0;
  int64_t* slot = nullptr;
  // staged gather: wait on stage_base + 4 * (stage_slot0 + piece of the
  // item's last source byte)
  uint64_t stage_base = 0;
  int64_t stage_slot0 = 0, stage_chunk = 0;
  // copy-engine relay: the slot comes from the item's last destination byte
  const RelaySlotFn* piece_slot = nullptr;
  const LoweredOp* op = nullptr;
};

void add_rect(std::vector<Tagged>& out, ItemSet& acc, uint64_t src, const std::vector<uint64_t>& dsts,
              const CopyRect& r, int64_t chunk, bool mc0, DeviceId src_dev, bool src_is_dst,
              RelayTags relay = {}) {
  const bool vec = ((src | static_cast<uint64_t>(r.src_off | r.dst_off | r.row_bytes | r.src_pitch | r.dst_pitch)) &
                    15) == 0 &&
                   std::all_of(dsts.begin(), dsts.end(), [](uint64_t d) { return (d & 15) == 0; });
  if (mc0 && !vec) throw rlplan::ValidationError("multicast copies must be 16-byte aligned");
  const int64_t unit = vec ? 16 : 2;
  const int64_t cap_units = std::min<int64_t>(chunk / unit, kMaxItemUnits);
  const int64_t row_units = r.row_bytes / unit;
  const int64_t sp = r.src_pitch / unit, dp = r.dst_pitch / unit;
  auto emit = [&](int64_t row0, int64_t col0, int64_t rows, int64_t cols) {
    CopyItem it;
    std::memset(&it, 0, sizeof(it));
    const int64_t src_begin = r.src_off + (row0 * sp + col0) * unit;
    it.src = src + static_cast<uint64_t>(src_begin);
    for (size_t j = 0; j < dsts.size(); ++j)
      it.dst[j] = dsts[j] + static_cast<uint64_t>(r.dst_off + (row0 * dp + col0) * unit);
    it.ndst = static_cast<uint16_t>(dsts.size());
    it.vec = static_cast<uint16_t>((vec ? kItemVec : 0) | (mc0 ? kItemMulticast0 : 0));
    it.row_units = static_cast<uint32_t>(cols);
    it.nrows = static_cast<uint32_t>(rows);
    it.src_pitch = static_cast<uint32_t>(rows > 1 ? sp : cols);
    it.dst_pitch = static_cast<uint32_t>(rows > 1 ? dp : cols);
    it.inv_row = 1.0f / static_cast<float>(cols);
    if (rows > 1 && ((rows - 1) * dp + cols >= (int64_t{1} << 32) || (rows - 1) * sp + cols >= (int64_t{1} << 32)))
      throw rlplan::ValidationError("copy item spans more than 2^32 units");
    if (relay.slot) {
      const uint64_t off = 4u * static_cast<uint64_t>((*relay.slot)++);
      if (relay.wait_base) it.wait_flag = relay.wait_base + off;
      if (relay.signal_base) it.signal_flag = relay.signal_base + off;
    }
    const int64_t src_end = src_begin + ((rows - 1) * sp + cols) * unit;
    if (relay.piece_slot) {
      const int64_t last = r.dst_off + ((row0 + rows - 1) * dp + col0 + cols) * unit - 1;
      const int64_t slot = (*relay.piece_slot)(relay.op, last);
      if (slot < 0) throw rlplan::ValidationError("fan-out bytes outside every relay piece");
      it.wait_flag = relay.stage_base + 4u * static_cast<uint64_t>(slot);
    } else if (relay.stage_base) {
      it.wait_flag = relay.stage_base + 4u * static_cast<uint64_t>(relay.stage_slot0 + (src_end - 1) / relay.stage_chunk);
    }
    out.push_back({it, src_dev, src_end, src_is_dst});
    const int64_t bytes = rows * cols * unit;
    acc.read += bytes;
    acc.written += bytes * static_cast<int64_t>(dsts.size());
  };
  if (row_units <= cap_units) {
    const int64_t rows_per = std::max<int64_t>(1, cap_units / std::max<int64_t>(row_units, 1));
    for (int64_t r0 = 0; r0 < r.rows; r0 += rows_per) emit(r0, 0, std::min(rows_per, r.rows - r0), row_units);
  } else {
    for (int64_t row = 0; row < r.rows; ++row)
      for (int64_t c0 = 0; c0 < row_units; c0 += cap_units) emit(row, c0, 1, std::min(cap_units, row_units - c0));
  }
}

uint64_t base_of(void* const* bufs, DeviceId d, const char* what) {
  if (!bufs) return 0;
  void* p = bufs[d];
  if (!p) throw rlplan::ValidationError(std::string("missing ") + what + " buffer for device " + std::to_string(d));
  return reinterpret_cast<uint64_t>(p);
}

}  // namespace

ItemSet build_items(const std::vector<Job>& jobs, int phase, const HostMap& hm, void* const* src_bufs,
                    void* const* dst_bufs, int64_t chunk_bytes, const std::vector<CeRun>* ce,
                    const CeSlotMap* ce_slots, const RelaySlotFn* relay_piece_slot) {
  ItemSet acc;
  std::vector<std::vector<Tagged>> streams;
  const bool accounting = src_bufs == nullptr;
  for (const auto& j : jobs) {
    if (j.phase != phase) continue;
    const uint64_t s = j.src_is_dst_buffer ? base_of(dst_bufs, j.src, "destination")
                                           : base_of(src_bufs, j.src, "source");
    for (size_t g = 0; g < j.dsts.size(); g += kMaxFan) {
      std::vector<uint64_t> dsts;
      std::vector<DeviceId> devs;  // parallel to dsts
      const bool mc0 = j.multicast && g == 0;
      for (size_t k = g; k < std::min(j.dsts.size(), g + kMaxFan); ++k) {
        devs.push_back(j.dsts[k]);
        if (mc0 && k == 0) {
          dsts.push_back(accounting ? 0 : j.mc_base);
          acc.remote_stores = true;
          continue;
        }
        dsts.push_back(base_of(dst_bufs, j.dsts[k], "destination"));
        if (hm.host[static_cast<size_t>(j.dsts[k])] != hm.me) acc.remote_stores = true;
      }
      streams.emplace_back();
      int64_t relay_slot = j.relay_base;
      if ((j.relay_wait || j.relay_signal) && j.dsts.size() > static_cast<size_t>(kMaxFan))
        throw rlplan::ValidationError("relay job with more than kMaxFan destinations");
      // Copy-engine runs / transport: plain jobs that read a real source shard
      const bool ce_job = ((ce && !ce->empty()) || hm.ce_remote) && plain_push(j, phase);
      std::vector<uint64_t> kept;
      for (CopyRect r : j.op->rects) {
        if (j.src_is_dst_buffer) {  // fan-out reads the leader's copy: destination geometry
          r.src_off = r.dst_off;
          r.src_pitch = r.dst_pitch;
        }
        const std::vector<uint64_t>* to = &dsts;
        if (ce_job) {
          kept.clear();
          for (size_t k = 0; k < dsts.size(); ++k) {
            if (hm.ce_remote && hm.host[static_cast<size_t>(devs[k])] != hm.me &&
                !hm.ce_sm_rects.count(std::make_tuple(j.src, devs[k], r.dst_off)))
              continue;
            if (ce && ce_covered(*ce, j.src, devs[k], r)) continue;
            kept.push_back(dsts[k]);
          }
          if (kept.empty()) continue;
          if (kept.size() != dsts.size()) to = &kept;
        }
        // Same-address copies (identical placement and buffers) are no-ops.
        if (!accounting && !mc0 && !j.relay_wait && !j.relay_signal && to->size() == 1 &&
            s + static_cast<uint64_t>(r.src_off) == (*to)[0] + static_cast<uint64_t>(r.dst_off))
          continue;
        if (j.relay_wait || j.relay_signal) {
          // relay pieces are cut at the slot granularity every rank agrees on
          const auto flags = [&](DeviceId d) {
            return accounting ? uint64_t{0} : hm.relay_flags.at(static_cast<size_t>(d));
          };
          RelayTags tags;
          tags.wait_base = j.relay_wait ? flags(j.src) : 0;
          tags.signal_base = j.relay_signal ? flags(j.dsts.front()) : 0;
          tags.slot = &relay_slot;
          add_rect(streams.back(), acc, s, dsts, r, hm.relay_chunk, mc0, j.src, j.src_is_dst_buffer, tags);
          continue;
        }
        if (j.ce_wait && j.ce_relay) {
          // wait for the relay piece holding the item's last leader byte
          // (pieces of one op land in order)
          if (relay_piece_slot == nullptr) throw rlplan::ValidationError("copy-engine relay without its slot map");
          RelayTags tags;
          tags.stage_base = accounting ? 4 : hm.ce_flags;
          tags.piece_slot = relay_piece_slot;
          tags.op = j.op;
          add_rect(streams.back(), acc, s, *to, r, chunk_bytes, mc0, j.src, j.src_is_dst_buffer, tags);
          continue;
        }
        if (j.ce_wait) {
          // wait for the transport copy that filled these leader bytes: the
          // item's rect lies inside one copy (copies carry whole rects)
          if (ce_slots == nullptr) throw rlplan::ValidationError("copy-engine star without its slot map");
          const int64_t slot = ce_slots->slot_of(j.op->src, j.src, r.dst_off);
          if (slot < 0) throw rlplan::ValidationError("fan-out rect not covered by a transport copy");
          RelayTags tags;
          tags.stage_base = accounting ? 4 : hm.ce_flags;  // every item of the rect waits on one slot
          tags.stage_slot0 = slot;
          tags.stage_chunk = int64_t{1} << 62;
          add_rect(streams.back(), acc, s, *to, r, chunk_bytes, mc0, j.src, j.src_is_dst_buffer, tags);
          continue;
        }
        if (hm.stage_chunk > 0 && phase == 0 && hm.host[static_cast<size_t>(j.src)] != hm.me) {
          RelayTags tags;  // reads a staging buffer: wait for the piece
          tags.stage_base = accounting ? 4 : hm.stage_flags;  // nonzero in accounting mode too
          tags.stage_slot0 = hm.stage_slot0.at(static_cast<size_t>(j.src));
          tags.stage_chunk = hm.stage_chunk;
          if (tags.stage_slot0 < 0) throw rlplan::ValidationError("staged source without slots");
          add_rect(streams.back(), acc, s, *to, r, chunk_bytes, mc0, j.src, j.src_is_dst_buffer, tags);
          continue;
        }
        add_rect(streams.back(), acc, s, *to, r, chunk_bytes, mc0, j.src, j.src_is_dst_buffer);
      }
    }
  }
  // Interleave the per-job streams round-robin so concurrently running CTAs
  // spread their stores over many destinations (NVLink ingress balance).
  // TMA-eligible items (16-byte, no multicast) first; the rest take the
  // LDG/STG kernel.
  //
  // With flag-synchronised (relay / star) items the whole phase runs in ONE
  // kernel, so local copies, pushes and per-chunk fan-outs overlap: the TMA
  // bulk kernel when every item is TMA-eligible, else the LDG/STG kernel
  // (two launches on one stream would serialise a wait behind the push it
  // needs on the other GPU). Deadlock freedom: within every round the items
  // that never wait come first, so when a CTA claims a waiting item of round
  // k every push of rounds <= k on this GPU is already claimed; the push it
  // waits for sits in round k of another GPU, whose waits in turn only depend
  // on our claimed pushes. A CTA never spins while holding unfinished
  // pushes, so every wait is eventually released.
  std::vector<const Tagged*> vec_items, other;
  size_t total = 0;
  bool flagged = false, all_tma = true;
  for (const auto& st : streams) {
    total += st.size();
    for (const auto& t : st) {
      flagged = flagged || t.it.wait_flag || t.it.signal_flag;
      all_tma = all_tma && t.it.vec == kItemVec;
    }
  }
  // HBM-only 1:1 phases are claimed job by job (each CTA walks consecutive
  // rows: contiguous read and write windows; the 7B back phase 4.72 -> 4.67
  // ms); broadcasts (fan-out >= 2) stay interleaved, which is faster for
  // them (forward 22.52 vs 22.31 ms; profiles/r02_order_sweep_n1.txt).
  // RR_ITEM_ORDER=rr|seq overrides the choice for sweeps.
  const char* order_env = std::getenv("RR_ITEM_ORDER");
  const bool one_to_one = acc.read > 0 && acc.written < acc.read + acc.read / 2;
  const bool sequential = !acc.remote_stores && !flagged &&
                          (order_env ? std::string(order_env) == "seq" : one_to_one);
  if (sequential) {
    for (const auto& st : streams)
      for (const auto& t : st) (t.it.vec == kItemVec ? vec_items : other).push_back(&t);
  } else
  for (size_t k = 0, seen = 0; seen < total; ++k)
    for (int waiting = 0; waiting < 2; ++waiting)
      for (const auto& st : streams)
        if (k < st.size() && (st[k].it.wait_flag != 0) == (waiting == 1)) {
          const bool tma = flagged ? all_tma : st[k].it.vec == kItemVec;
          (tma ? vec_items : other).push_back(&st[k]);
          ++seen;
        }
  if (hm.stage_chunk > 0) {
    // staged gather: items that can run now first, then the staged ones in
    // the order their pieces arrive (slot order)
    for (auto* list : {&vec_items, &other}) {
      std::stable_sort(list->begin(), list->end(), [](const Tagged* a, const Tagged* b) {
        return a->it.wait_flag < b->it.wait_flag;  // 0 (no wait) first
      });
    }
  } else if ((ce_slots != nullptr && !ce_slots->ready.empty()) || relay_piece_slot != nullptr) {
    // copy-engine star / relay: items that can run now first, then the
    // fan-out items in the order their copies or pieces land (a CTA spinning
    // on a late copy must not hold up items whose copy is already in); relay
    // pieces (slots after the star's) in slot order
    const uint64_t base = accounting ? 4 : hm.ce_flags;
    auto ready = [&](const Tagged* t) {
      if (!t->it.wait_flag) return -1.0;
      const size_t slot = static_cast<size_t>((t->it.wait_flag - base) / 4);
      if (ce_slots != nullptr && slot < ce_slots->ready.size()) return ce_slots->ready[slot];
      return 1e20 + static_cast<double>(slot);
    };
    for (auto* list : {&vec_items, &other})
      std::stable_sort(list->begin(), list->end(), [&](const Tagged* a, const Tagged* b) { return ready(a) < ready(b); });
  }
  acc.n_vec = static_cast<int>(vec_items.size());
  vec_items.insert(vec_items.end(), other.begin(), other.end());
  if (vec_items.size() >= (size_t{1} << 31)) throw rlplan::ValidationError("too many copy items");
  acc.items.reserve(vec_items.size());
  for (const Tagged* t : vec_items) {
    acc.items.push_back(t->it);
    acc.src_dev.push_back(t->src_dev);
    acc.src_end.push_back(t->src_end);
    acc.src_is_dst.push_back(t->src_is_dst);
  }
  return acc;
}

namespace {

// Longest arithmetic chain of unused copies starting at i: copy k of the
// chain sits at (src_off, dst_off) + k * (ds, dd). Candidates are the same
// shape, sorted by src_off; ok(ds, dd) says whether a stride pair can be
// expressed (non-overlapping rows, pitch limits, 3D divisibility).
template <class Ok>
std::vector<size_t> best_chain(const std::vector<CeCopy>& c, const std::vector<bool>& used, size_t i, Ok ok) {
  std::map<std::pair<int64_t, int64_t>, size_t> at;  // (src_off, dst_off) -> index
  for (size_t k = i; k < c.size(); ++k)
    if (!used[k]) at.emplace(std::make_pair(c[k].src_off, c[k].dst_off), k);
  std::vector<size_t> best{i};
  size_t tried = 0;
  for (size_t j = i + 1; j < c.size() && tried < 64; ++j) {
    if (used[j]) continue;
    ++tried;
    const int64_t ds = c[j].src_off - c[i].src_off, dd = c[j].dst_off - c[i].dst_off;
    if (ds <= 0 || dd <= 0 || !ok(ds, dd)) continue;
    std::vector<size_t> chain{i, j};
    for (;;) {
      const auto it = at.find({c[i].src_off + ds * static_cast<int64_t>(chain.size()),
                               c[i].dst_off + dd * static_cast<int64_t>(chain.size())});
      if (it == at.end()) break;
      chain.push_back(it->second);
    }
    if (chain.size() > best.size()) best = std::move(chain);
  }
  return best;
}

// Merge the elementary copies of one (source, destination) pair.
std::vector<CeCopy> merge_pair(std::vector<CeCopy> flat, std::vector<CeCopy> strided, int64_t max_pitch) {
  std::vector<CeCopy> out;
  // contiguous pieces: coalesce neighbours, then chain equal widths into 2D
  std::sort(flat.begin(), flat.end(), [](const CeCopy& a, const CeCopy& b) { return a.src_off < b.src_off; });
  std::vector<CeCopy> co;
  for (const auto& c : flat) {
    if (!co.empty() && co.back().src_off + co.back().width == c.src_off &&
        co.back().dst_off + co.back().width == c.dst_off)
      co.back().width += c.width;
    else
      co.push_back(c);
  }
  std::map<int64_t, std::vector<CeCopy>> by_width;
  for (const auto& c : co) by_width[c.width].push_back(c);
  for (auto& [w, list] : by_width) {
    std::vector<bool> used(list.size(), false);
    for (size_t i = 0; i < list.size(); ++i) {
      if (used[i]) continue;
      const auto chain = best_chain(list, used, i, [&, w = w](int64_t ds, int64_t dd) {
        return ds >= w && dd >= w && ds <= max_pitch && dd <= max_pitch;
      });
      for (size_t k : chain) used[k] = true;
      CeCopy m = list[i];
      if (chain.size() > 1) {
        m.height = static_cast<int64_t>(chain.size());
        m.src_pitch = list[chain[1]].src_off - list[i].src_off;
        m.dst_pitch = list[chain[1]].dst_off - list[i].dst_off;
      } else {
        m.src_pitch = m.dst_pitch = m.width;
      }
      out.push_back(m);
    }
  }
  // row-parallel pieces: chain equal shapes into 3D
  using Shape = std::tuple<int64_t, int64_t, int64_t, int64_t>;
  std::map<Shape, std::vector<CeCopy>> by_shape;
  for (const auto& c : strided) by_shape[{c.width, c.height, c.src_pitch, c.dst_pitch}].push_back(c);
  for (auto& [shape, list] : by_shape) {
    std::sort(list.begin(), list.end(), [](const CeCopy& a, const CeCopy& b) { return a.src_off < b.src_off; });
    std::vector<bool> used(list.size(), false);
    const auto [w, h, sp, dp] = shape;
    for (size_t i = 0; i < list.size(); ++i) {
      if (used[i]) continue;
      const auto chain = best_chain(list, used, i, [&, h = h, sp = sp, dp = dp](int64_t ds, int64_t dd) {
        return ds % sp == 0 && dd % dp == 0 && ds / sp >= h && dd / dp >= h;
      });
      for (size_t k : chain) used[k] = true;
      CeCopy m = list[i];
      if (chain.size() > 1) {
        m.depth = static_cast<int64_t>(chain.size());
        m.src_slice = list[chain[1]].src_off - list[i].src_off;
        m.dst_slice = list[chain[1]].dst_off - list[i].dst_off;
      }
      out.push_back(m);
    }
  }
  std::sort(out.begin(), out.end(), [](const CeCopy& a, const CeCopy& b) { return a.dst_off < b.dst_off; });
  return out;
}

}  // namespace

std::vector<CeCopy> ce_copies_of(const std::vector<LoweredOp>& ops, const HostMap& hm, int g, int64_t max_pitch) {
  HostMap h = hm;
  h.me = g;
  h.ce_remote = true;
  h.ce_star = false;
  h.relay_flags.clear();
  h.mc.clear();
  h.stage_chunk = 0;
  return ce_transport_copies(build_jobs(ops, h, 0), h, max_pitch);
}

namespace {
std::vector<int> host_ids(const HostMap& hm) {
  std::vector<int> hosts(hm.host.begin(), hm.host.end());
  hosts.push_back(hm.me);
  std::sort(hosts.begin(), hosts.end());
  hosts.erase(std::unique(hosts.begin(), hosts.end()), hosts.end());
  return hosts;
}

bool copy_has(const CeCopy& c, int64_t off) {
  int64_t rel = off - c.dst_off;
  if (rel < 0) return false;
  if (c.depth > 1) {
    const int64_t z = rel / c.dst_slice;
    if (z >= c.depth) return false;
    rel -= z * c.dst_slice;
  }
  if (c.height > 1) {
    const int64_t y = rel / c.dst_pitch;
    if (y >= c.height) return false;
    rel -= y * c.dst_pitch;
  }
  return rel < c.width;
}
}  // namespace

std::vector<bool> star_flagged(const std::vector<CeCopy>& copies, const HostMap& hm) {
  std::vector<bool> out(copies.size(), false);
  int64_t run = 0;
  for (size_t k = 0; k < copies.size(); ++k) {
    run += copies[k].bytes();
    const bool last_to_receiver = k + 1 == copies.size() || hm.host[static_cast<size_t>(copies[k + 1].dst)] !=
                                                                 hm.host[static_cast<size_t>(copies[k].dst)];
    if (run >= kStarFlagBytes || last_to_receiver) {
      out[k] = true;
      run = 0;
    }
  }
  return out;
}

CeSlotMap ce_slot_map(const std::vector<LoweredOp>& ops, const HostMap& hm, int h, int64_t max_pitch) {
  CeSlotMap m;
  int64_t slot = 0;
  std::map<int, std::vector<CeCopy>> of;
  for (int g : host_ids(hm)) {
    if (g == h) continue;
    of[g] = ce_copies_of(ops, hm, g, max_pitch);
    const auto flagged = star_flagged(of[g], hm);
    // a copy's items wait on the slot of the flagged copy that ends its group
    std::vector<size_t> mine;
    for (size_t k = 0; k < of[g].size(); ++k)
      if (hm.host[static_cast<size_t>(of[g][k].dst)] == h) mine.push_back(k);
    const size_t first = m.copies.size();
    for (size_t k : mine) m.copies.push_back({of[g][k], slot++});
    int64_t wait = -1;
    for (size_t i = mine.size(); i-- > 0;) {
      if (flagged[mine[i]]) wait = m.copies[first + i].second;
      m.copies[first + i].second = wait;
    }
  }
  // landing times: each transfer into h from its simulated start, copy by copy
  m.ready.assign(m.copies.size(), 0.0);
  std::map<int, int64_t> first_slot;  // sender -> slot of its first copy to h
  for (size_t i = 0; i < m.copies.size(); ++i)  // a sender's copies to h are consecutive (one transfer)
    first_slot.emplace(hm.host[static_cast<size_t>(m.copies[i].first.src)], static_cast<int64_t>(i));
  for (const auto& t : ce_schedule(ops, hm, max_pitch)) {
    if (t.receiver != h) continue;
    double at = t.start;
    const int64_t s0 = first_slot[t.sender];
    for (size_t k = 0; k < t.count; ++k) {
      at += static_cast<double>(of[t.sender][t.first + k].bytes()) / 775e9;
      m.ready[static_cast<size_t>(s0) + k] = at;
    }
  }
  return m;
}

int64_t CeSlotMap::slot_of(DeviceId src, DeviceId dst, int64_t dst_off) const {
  for (const auto& [c, slot] : copies)
    if (c.src == src && c.dst == dst && copy_has(c, dst_off)) return slot;
  return -1;
}

int64_t ce_star_slots(const std::vector<LoweredOp>& ops, const HostMap& hm, int h, int64_t max_pitch) {
  return static_cast<int64_t>(ce_slot_map(ops, hm, h, max_pitch).copies.size());
}

std::vector<int64_t> ce_send_slots(const std::vector<LoweredOp>& ops, const HostMap& hm,
                                   const std::vector<CeCopy>& mine, int64_t max_pitch) {
  std::map<int, int64_t> base;  // receiver -> slots taken by lower-id senders
  for (int h : host_ids(hm)) {
    if (h == hm.me) continue;
    int64_t n = 0;
    for (int g : host_ids(hm)) {
      if (g == h) continue;
      if (g == hm.me) break;
      for (const auto& c : ce_copies_of(ops, hm, g, max_pitch))
        if (hm.host[static_cast<size_t>(c.dst)] == h) ++n;
    }
    base[h] = n;
  }
  std::vector<int64_t> out;
  for (const auto& c : mine) out.push_back(base[hm.host[static_cast<size_t>(c.dst)]]++);
  return out;
}

std::vector<CeCopy> ce_transport_copies(const std::vector<Job>& jobs, const HostMap& hm, int64_t max_pitch,
                                        std::set<std::tuple<DeviceId, DeviceId, int64_t>>* sm_rects) {
  std::map<std::pair<DeviceId, DeviceId>, std::pair<std::vector<CeCopy>, std::vector<CeCopy>>> pairs;
  for (const auto& j : jobs) {
    if (!plain_push(j, j.phase) || hm.host[static_cast<size_t>(j.src)] != hm.me) continue;
    if (ce_relay_op(*j.op, hm)) continue;  // travels by the relay
    for (DeviceId d : j.dsts) {
      if (hm.host[static_cast<size_t>(d)] == hm.me) continue;
      auto& [flat, strided] = pairs[{j.src, d}];
      for (const auto& r : j.op->rects) {
        CeCopy c;
        c.src = j.src;
        c.dst = d;
        c.src_off = r.src_off;
        c.dst_off = r.dst_off;
        if (r.rows == 1 || (r.src_pitch == r.row_bytes && r.dst_pitch == r.row_bytes)) {
          c.width = r.row_bytes * r.rows;
          flat.push_back(c);
        } else {
          c.width = r.row_bytes;
          c.height = r.rows;
          c.src_pitch = r.src_pitch;
          c.dst_pitch = r.dst_pitch;
          c.strided = true;
          strided.push_back(c);
        }
      }
    }
  }
  // rotation rounds over the hosts (ascending ids)
  std::vector<int> hosts(hm.host.begin(), hm.host.end());
  hosts.push_back(hm.me);
  std::sort(hosts.begin(), hosts.end());
  hosts.erase(std::unique(hosts.begin(), hosts.end()), hosts.end());
  const int H = static_cast<int>(hosts.size());
  const int pos = static_cast<int>(std::find(hosts.begin(), hosts.end(), hm.me) - hosts.begin());
  std::vector<CeCopy> out;
  for (int r = 1; r < H; ++r) {
    const int h = hosts[static_cast<size_t>((pos + r) % H)];
    for (auto& [sd, lists] : pairs) {
      if (hm.host[static_cast<size_t>(sd.second)] != h) continue;
      auto merged = merge_pair(std::move(lists.first), std::move(lists.second), max_pitch);
      for (const auto& c : merged) {
        if (hm.ce_hybrid && c.strided && c.depth == 1) {
          if (sm_rects) sm_rects->insert({c.src, c.dst, c.dst_off});  // an unmerged row-parallel rect
          continue;
        }
        out.push_back(c);
      }
    }
  }
  return out;
}

std::vector<CeTransfer> ce_schedule(const std::vector<LoweredOp>& ops, const HostMap& hm, int64_t max_pitch) {
  constexpr double kRate = 775e9;                   // copy-engine payload rate per GPU, pairwise (r02 probes)
  constexpr double kCopy = 4e-6, kCopy2d = 10e-6;  // per submission (2D copies cost more)
  const std::vector<int> hosts = host_ids(hm);
  const int H = static_cast<int>(hosts.size());
  std::map<int, int> pos;
  for (int i = 0; i < H; ++i) pos[hosts[static_cast<size_t>(i)]] = i;
  std::map<int, std::vector<CeCopy>> copies;
  std::map<int, int64_t> base;  // first schedule slot of each host
  for (int g : hosts) copies[g] = ce_copies_of(ops, hm, g, max_pitch);
  for (int h : hosts) {
    int64_t incoming = 0;
    for (int g : hosts)
      if (g != h)
        for (const auto& c : copies[g]) incoming += hm.host[static_cast<size_t>(c.dst)] == h;
    base[h] = incoming;
  }
  // Transfers: each sender's copies to one receiver (its rotation round
  // r = receiver position - sender position, mod H; ce_transport_copies
  // already issues them in round order).
  std::vector<CeTransfer> all;
  std::vector<int> round;
  std::vector<double> dur;
  for (int g : hosts) {
    const auto& cs = copies[g];
    for (size_t k = 0; k < cs.size();) {
      CeTransfer t;
      t.sender = g;
      t.receiver = hm.host[static_cast<size_t>(cs[k].dst)];
      t.first = k;
      double d = 0;
      while (k < cs.size() && hm.host[static_cast<size_t>(cs[k].dst)] == t.receiver) {
        d += static_cast<double>(cs[k].bytes()) / kRate + (cs[k].height > 1 && cs[k].depth == 1 ? kCopy2d : kCopy);
        ++k;
      }
      t.count = k - t.first;
      all.push_back(t);
      round.push_back((pos[t.receiver] - pos[g] + H) % H);
      dur.push_back(d);
    }
  }
  // Candidate orders, simulated at the measured rates (a transfer starts
  // when its sender is free and its receiver has finished the transfer
  // before it in that receiver's order); the shortest makespan wins:
  //   rounds: every sender in rotation order, each receiver served in round
  //           order (the rounds stay aligned without a barrier: all-to-all);
  //   greedy: list schedule, next the transfer that can start first (ties:
  //           the sender with the most work left) — sparse patterns where
  //           rotation rounds leave receivers idle (70B at 8 GPUs).
  const size_t T = all.size();
  std::map<int, double> load;
  for (size_t i = 0; i < T; ++i) load[all[i].sender] += dur[i];
  struct Sim {
    std::vector<double> start, end;
    std::vector<size_t> order;  // issue order (ascending start)
    double makespan = 0;
  };
  auto run = [&](bool rounds) {
    Sim sim;
    sim.start.assign(T, 0);
    sim.end.assign(T, 0);
    std::map<int, double> free_s, free_r, left = load;
    std::vector<bool> done(T, false);
    for (size_t n = 0; n < T; ++n) {
      size_t best = T;
      double bs = 0;
      for (size_t i = 0; i < T; ++i) {
        if (done[i]) continue;
        if (rounds) {  // strictly by round, then sender: the receiver order is the round order
          if (best == T || round[i] < round[best] || (round[i] == round[best] && all[i].sender < all[best].sender))
            best = i;
          continue;
        }
        const double st = std::max(free_s[all[i].sender], free_r[all[i].receiver]);
        if (best == T || st < bs - 1e-9 ||
            (st < bs + 1e-9 && left[all[i].sender] > left[all[best].sender] + 1e-12)) {
          best = i;
          bs = st;
        }
      }
      const CeTransfer& t = all[best];
      sim.start[best] = std::max(free_s[t.sender], free_r[t.receiver]);
      sim.end[best] = sim.start[best] + dur[best];
      free_s[t.sender] = free_r[t.receiver] = sim.end[best];
      left[t.sender] -= dur[best];
      done[best] = true;
      sim.order.push_back(best);
      sim.makespan = std::max(sim.makespan, sim.end[best]);
    }
    return sim;
  };
  const Sim a = run(true), g = run(false);
  const Sim& pick = g.makespan < a.makespan * 0.99 ? g : a;
  // Receiver chains in the chosen order: each transfer into a host waits for
  // the one before it (unless the same sender: stream order); every wait
  // points to an earlier-issued transfer, so no cycles.
  std::map<int, int64_t> waits;  // sender -> slots handed out
  std::map<int, size_t> last_into;
  for (size_t i : pick.order) {
    CeTransfer& t = all[i];
    t.start = pick.start[i];
    t.end = pick.end[i];
    const auto prev = last_into.find(t.receiver);
    if (prev != last_into.end() && all[prev->second].sender != t.sender) {
      t.wait_slot = base[t.sender] + waits[t.sender]++;
      all[prev->second].signal_host = t.sender;
      all[prev->second].signal_slot = t.wait_slot;
    }
    last_into[t.receiver] = i;
  }
  // each sender issues its transfers in the chosen order
  std::vector<CeTransfer> out;
  for (size_t i : pick.order) out.push_back(all[i]);
  std::stable_sort(out.begin(), out.end(), [](const CeTransfer& a, const CeTransfer& b) { return a.sender < b.sender; });
  return out;
}

int64_t ce_relay_base(const std::vector<LoweredOp>& ops, const HostMap& hm, int h, int64_t max_pitch) {
  int64_t n = ce_star_slots(ops, hm, h, max_pitch);
  for (const auto& t : ce_schedule(ops, hm, max_pitch))
    if (t.sender == h && t.wait_slot >= 0) n = std::max(n, t.wait_slot + 1);
  return n;
}

int64_t ce_flag_slots(const std::vector<LoweredOp>& ops, const HostMap& hm, int h, int64_t max_pitch) {
  int64_t n = ce_relay_base(ops, hm, h, max_pitch);
  if (hm.ce_relay)
    for (const auto& r : ce_relay_ops(ops, hm)) n += static_cast<int64_t>(r.pieces.size());
  return n;
}

bool ce_relay_op(const LoweredOp& op, const HostMap& hm) {
  if (!hm.ce_relay || !hm.hierarchical) return false;
  const int hs = hm.host[static_cast<size_t>(op.src)];
  std::set<int> remote;
  for (DeviceId d : op.dst)
    if (hm.host[static_cast<size_t>(d)] != hs) remote.insert(hm.host[static_cast<size_t>(d)]);
  return remote.size() >= 2;
}

std::vector<CeRelayOp> ce_relay_ops(const std::vector<LoweredOp>& ops, const HostMap& hm) {
  std::vector<CeRelayOp> out;
  int64_t slot = 0;
  // RR_RELAY_PIECE_MIB overrides the piece size for sweeps (identical on every rank)
  const char* env = std::getenv("RR_RELAY_PIECE_MIB");
  const int64_t kRelayPieceBytes = env ? std::max<int64_t>(1, std::atoll(env)) << 20 : rr::kRelayPieceBytes;
  for (const auto& op : ops) {
    if (!ce_relay_op(op, hm)) continue;
    CeRelayOp r;
    r.op = &op;
    r.src_host = hm.host[static_cast<size_t>(op.src)];
    const auto groups = by_host(op, hm);
    r.chain = relay_chain(groups, r.src_host);
    for (int h : r.chain) r.leader.push_back(groups.at(h).front());
    // pieces: rects cut into <= kRelayPieceBytes row ranges; neighbouring 1D
    // pieces contiguous on both sides are coalesced
    for (const auto& rc : op.rects) {
      const bool flat = rc.rows == 1 || (rc.src_pitch == rc.row_bytes && rc.dst_pitch == rc.row_bytes);
      if (flat) {
        const int64_t total = rc.row_bytes * rc.rows;
        for (int64_t off = 0; off < total; off += kRelayPieceBytes) {
          const int64_t w = std::min(kRelayPieceBytes, total - off);
          auto& v = r.pieces;
          if (!v.empty() && v.back().height == 1 && v.back().src_off + v.back().width == rc.src_off + off &&
              v.back().dst_off + v.back().width == rc.dst_off + off && v.back().width + w <= kRelayPieceBytes) {
            v.back().width += w;
            continue;
          }
          CeRelayPiece p;
          p.src_off = rc.src_off + off;
          p.dst_off = rc.dst_off + off;
          p.width = w;
          v.push_back(p);
        }
      } else {
        const int64_t per = std::max<int64_t>(1, kRelayPieceBytes / rc.row_bytes);
        for (int64_t row = 0; row < rc.rows; row += per) {
          CeRelayPiece p;
          p.src_off = rc.src_off + row * rc.src_pitch;
          p.dst_off = rc.dst_off + row * rc.dst_pitch;
          p.width = rc.row_bytes;
          p.height = std::min(per, rc.rows - row);
          p.src_pitch = rc.src_pitch;
          p.dst_pitch = rc.dst_pitch;
          r.pieces.push_back(p);
        }
      }
    }
    r.slot0 = slot;
    slot += static_cast<int64_t>(r.pieces.size());
    out.push_back(std::move(r));
  }
  return out;
}

}  // namespace rr
