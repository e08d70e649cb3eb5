// Executor work construction (see exec_plan.hpp). The upstream runtime
// broadcasts each TP partition from its chosen source to every destination
// (PAPER.md:515); here a payload crosses NVLink once per destination host
// and is replicated inside the host from HBM.
#include "exec_plan.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>

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

}  // namespace

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
  for (const auto& op : ops) {
    const int hs = hm.host[static_cast<size_t>(op.src)];
    const auto groups = by_host(op, hm);
    const auto mine = groups.find(hm.me);
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
        for (const auto& [h, list] : groups) {
          Job j;
          j.phase = 0;
          j.src = op.src;
          j.op = &op;
          if (h == hm.me)
            j.dsts = list;
          else
            j.dsts = {list.front()};
          jobs.push_back(std::move(j));
        }
      }
    } else if (mine != groups.end()) {  // pull: each destination host fetches for itself
      Job j;
      j.phase = 0;
      j.src = op.src;
      j.op = &op;
      j.dsts = hs == hm.me ? mine->second : std::vector<DeviceId>{mine->second.front()};
      jobs.push_back(std::move(j));
    }
    if (hs != hm.me && mine != groups.end() && mine->second.size() > 1) {
      Job j;
      j.phase = 1;
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

namespace {

// An item plus where it reads from (for onload pipelining).
struct Tagged {
  CopyItem it;
  DeviceId src_dev;
  int64_t src_end;
  bool src_is_dst;
};

// Chunk one rectangle for (src base, dst bases) into items.
void add_rect(std::vector<Tagged>& out, ItemSet& acc, uint64_t src, const std::vector<uint64_t>& dsts,
              const CopyRect& r, int64_t chunk, bool mc0, DeviceId src_dev, bool src_is_dst) {
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
    out.push_back({it, src_dev, src_begin + ((rows - 1) * sp + cols) * unit, src_is_dst});
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
                    void* const* dst_bufs, int64_t chunk_bytes) {
  ItemSet acc;
  std::vector<std::vector<Tagged>> streams;
  const bool accounting = src_bufs == nullptr;
  for (const auto& j : jobs) {
    if (j.phase != phase) continue;
    const uint64_t s = j.src_is_dst_buffer ? base_of(dst_bufs, j.src, "destination")
                                           : base_of(src_bufs, j.src, "source");
    for (size_t g = 0; g < j.dsts.size(); g += kMaxFan) {
      std::vector<uint64_t> dsts;
      const bool mc0 = j.multicast && g == 0;
      for (size_t k = g; k < std::min(j.dsts.size(), g + kMaxFan); ++k) {
        if (mc0 && k == 0) {
          dsts.push_back(accounting ? 0 : j.mc_base);
          acc.remote_stores = true;
          continue;
        }
        dsts.push_back(base_of(dst_bufs, j.dsts[k], "destination"));
        if (hm.host[static_cast<size_t>(j.dsts[k])] != hm.me) acc.remote_stores = true;
      }
      streams.emplace_back();
      for (CopyRect r : j.op->rects) {
        if (j.src_is_dst_buffer) {  // fan-out reads the leader's copy: destination geometry
          r.src_off = r.dst_off;
          r.src_pitch = r.dst_pitch;
        }
        // Same-address copies (identical placement and buffers) are no-ops.
        if (!accounting && !mc0 && dsts.size() == 1 &&
            s + static_cast<uint64_t>(r.src_off) == dsts[0] + static_cast<uint64_t>(r.dst_off))
          continue;
        add_rect(streams.back(), acc, s, dsts, r, chunk_bytes, mc0, j.src, j.src_is_dst_buffer);
      }
    }
  }
  // Interleave the per-job streams round-robin so concurrently running CTAs
  // spread their stores over many destinations (NVLink ingress balance).
  // TMA-eligible items (16-byte, no multicast) first; the rest take the
  // LDG/STG kernel.
  std::vector<const Tagged*> vec_items, other;
  size_t total = 0;
  for (const auto& st : streams) total += st.size();
  for (size_t k = 0, seen = 0; seen < total; ++k)
    for (const auto& st : streams)
      if (k < st.size()) {
        (st[k].it.vec == kItemVec ? vec_items : other).push_back(&st[k]);
        ++seen;
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

}  // namespace rr
