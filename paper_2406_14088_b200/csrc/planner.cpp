// Reallocation planner and lowering.
//
// plan_param_realloc restates SPEC.md:569-577 with the design decisions of
// SPEC.md:594-598 and the hierarchical procedure of PAPER.md:500 and
// PAPER.md:515 (outer loop over stage pairs with common layers, inner loop
// over destination GPUs, cheapest source wins, sources broadcast in
// parallel). lower_plan turns each (src, payload) into 2D copy rectangles by
// intersecting the payload's logical slices with the source and destination
// shard layouts (layout.cpp), which is what the sm_100a kernels execute.
#include <algorithm>
#include <cstdio>
#include <map>
#include <sstream>
#include <tuple>

#include "rlplan/realloc.hpp"

namespace rlplan {

std::vector<std::pair<Count, Count>> stage_layer_map(Count num_layers, int pp) {
  if (pp < 1) throw ValidationError("stage_layer_map: pp must be >= 1");
  if (pp > num_layers) throw ValidationError("stage_layer_map: pp must not exceed num_layers");
  std::vector<std::pair<Count, Count>> stages;
  stages.reserve(static_cast<size_t>(pp));
  const Count base = num_layers / pp, extra = num_layers % pp;
  Count start = 0;
  for (int s = 0; s < pp; ++s) {
    const Count len = base + (s < extra ? 1 : 0);
    stages.emplace_back(start, start + len);
    start += len;
  }
  return stages;
}

namespace {

// Extended layer range of stage s: stage 0 also holds the embedding (-1),
// the last stage also holds the final norm + head (L).
std::pair<Count, Count> ext_range(const std::vector<std::pair<Count, Count>>& stages, int s,
                                  Count L) {
  const int last = static_cast<int>(stages.size()) - 1;
  Count lo = stages[static_cast<size_t>(s)].first, hi = stages[static_cast<size_t>(s)].second;
  if (s == 0) lo = -1;
  if (s == last) hi = L + 1;
  return {lo, hi};
}

bool is_kv(const LogicalTensor& t) { return t.kind == kK || t.kind == kV; }

// Whether tensor t belongs to a payload of the given kind (G5, G6).
bool in_payload(const LogicalTensor& t, bool replicated, int part) {
  const bool rep = t.split == SplitKind::Replicated;
  if (rep != replicated) return false;
  if (rep) return true;
  return part == kPartAll || (part == kPartKv) == is_kv(t);
}

Bytes range_bytes(const std::vector<LogicalTensor>& inv, const ModelSpec& m, Count lo, Count hi,
                  bool replicated, Count degree, int part = kPartAll) {
  Bytes n = 0;
  for (const auto& t : inv) {
    if (t.ext_layer < lo || t.ext_layer >= hi) continue;
    if (!in_payload(t, replicated, part)) continue;
    n += t.rows * t.cols / (replicated ? 1 : degree);
  }
  return n * m.param_bytes;
}

using OpKey = std::tuple<DeviceId, Count, Count, int, int, bool, int>;

OpKey key_of(DeviceId src, const ShardDescriptor& p) {
  return {src, p.layer_start, p.layer_end, p.tp_rank, p.tp_degree, p.replicated, p.part};
}

}  // namespace

Bytes payload_bytes(const ModelSpec& model, const ShardDescriptor& p) {
  const auto inv = tensor_inventory(model);
  return range_bytes(inv, model, p.layer_start, p.layer_end, p.replicated, p.tp_degree, p.part);
}

ReallocPlan plan_param_realloc(const ModelSpec& m, const Placement& src, const Placement& dst,
                               const ClusterSpec& cluster, SourcePolicy policy) {
  cluster.validate();
  validate_placement(m, src, cluster);
  validate_placement(m, dst, cluster);
  const auto inv = tensor_inventory(m);
  const Count L = m.num_layers;
  const int tp1 = src.strategy.tp, tp2 = dst.strategy.tp;
  const int G = static_cast<int>(lcm_count(tp1, tp2));
  // K/V as their own payloads when either side replicates KV heads (G6).
  const int e1 = kv_degree(m, src), e2 = kv_degree(m, dst);
  const bool kv_class = e1 != tp1 || e2 != tp2;
  const int Gkv = static_cast<int>(lcm_count(e1, e2));
  const int split_part = kv_class ? kPartNoKv : kPartAll;
  for (const auto& t : inv) {
    if (kv_class && is_kv(t)) {
      if (t.rows % Gkv)
        throw ValidationError("plan_param_realloc: lcm(kv slices) must divide the k/v rows");
      continue;
    }
    if (t.split == SplitKind::Rows && t.rows % G)
      throw ValidationError("plan_param_realloc: lcm(tp) must divide every row-split dimension");
    if (t.split == SplitKind::Cols && t.cols % G)
      throw ValidationError("plan_param_realloc: lcm(tp) must divide every column-split dimension");
  }
  const auto s_stages = stage_layer_map(L, src.strategy.pp);
  const auto d_stages = stage_layer_map(L, dst.strategy.pp);

  ReallocPlan plan;
  std::map<OpKey, size_t> remote_index, local_index;
  std::map<DeviceId, Bytes> egress;  // bytes assigned per source (balanced policy)

  auto emit = [&](DeviceId s, DeviceId d, const ShardDescriptor& payload, Bytes bytes) {
    const bool local = s == d;
    auto& index = local ? local_index : remote_index;
    auto& list = local ? plan.local_ops : plan.ops;
    const OpKey key = key_of(s, payload);
    auto it = index.find(key);
    if (it == index.end()) {
      it = index.emplace(key, list.size()).first;
      list.push_back(BroadcastOp{s, {}, payload, bytes});
    }
    list[it->second].dst.push_back(d);
  };

  // Cheapest holder for destination d: self, then the highest
  // bandwidth class; ties broken by policy.
  auto choose = [&](const std::vector<DeviceId>& holders, DeviceId d, Bytes bytes) {
    if (std::find(holders.begin(), holders.end(), d) != holders.end()) return d;
    double best_bw = -1;
    for (DeviceId h : holders) best_bw = std::max(best_bw, link_bandwidth(cluster, h, d));
    DeviceId pick = -1;
    for (DeviceId h : holders) {  // holders ascending
      if (link_bandwidth(cluster, h, d) != best_bw) continue;
      if (pick < 0) {
        pick = h;
        if (policy == SourcePolicy::Spec) break;
        continue;
      }
      if (egress[h] < egress[pick]) pick = h;
    }
    egress[pick] += bytes;
    return pick;
  };

  for (int i = 0; i < src.strategy.pp; ++i) {
    const auto si = ext_range(s_stages, i, L);
    for (int j = 0; j < dst.strategy.pp; ++j) {
      const auto dj = ext_range(d_stages, j, L);
      const Count lo = std::max(si.first, dj.first), hi = std::min(si.second, dj.second);
      if (lo >= hi) continue;
      const Bytes split_bytes = range_bytes(inv, m, lo, hi, false, G, split_part);
      const Bytes kv_bytes = kv_class ? range_bytes(inv, m, lo, hi, false, Gkv, kPartKv) : 0;
      const Bytes rep_bytes = range_bytes(inv, m, lo, hi, true, 1);
      std::vector<DeviceId> all_src;
      for (int dp = 0; dp < src.strategy.dp; ++dp)
        for (int tp = 0; tp < tp1; ++tp) all_src.push_back(device_at(src, cluster, i, dp, tp));
      std::sort(all_src.begin(), all_src.end());
      for (int dp = 0; dp < dst.strategy.dp; ++dp) {
        for (int tr = 0; tr < tp2; ++tr) {
          const DeviceId d = device_at(dst, cluster, j, dp, tr);
          if (split_bytes > 0) {
            for (int k = tr * (G / tp2); k < (tr + 1) * (G / tp2); ++k) {
              std::vector<DeviceId> holders;
              for (int sdp = 0; sdp < src.strategy.dp; ++sdp)
                holders.push_back(device_at(src, cluster, i, sdp, k / (G / tp1)));
              std::sort(holders.begin(), holders.end());
              const ShardDescriptor payload{lo, hi, k, G, false, split_part};
              emit(choose(holders, d, split_bytes), d, payload, split_bytes);
            }
          }
          if (kv_bytes > 0) {
            // K/V slices of this rank's head range; every source TP rank
            // whose kv slice covers k holds it (replicas included).
            const int s2 = tr * e2 / tp2;
            for (int k = s2 * (Gkv / e2); k < (s2 + 1) * (Gkv / e2); ++k) {
              const int q = k / (Gkv / e1);
              std::vector<DeviceId> holders;
              for (int sdp = 0; sdp < src.strategy.dp; ++sdp)
                for (int st = q * (tp1 / e1); st < (q + 1) * (tp1 / e1); ++st)
                  holders.push_back(device_at(src, cluster, i, sdp, st));
              std::sort(holders.begin(), holders.end());
              const ShardDescriptor payload{lo, hi, k, Gkv, false, kPartKv};
              emit(choose(holders, d, kv_bytes), d, payload, kv_bytes);
            }
          }
          if (rep_bytes > 0) {
            const ShardDescriptor payload{lo, hi, 0, 1, true};
            emit(choose(all_src, d, rep_bytes), d, payload, rep_bytes);
          }
        }
      }
    }
  }

  std::map<DeviceId, Seconds> busy;
  for (const auto& op : plan.ops) {
    double bw = local_bandwidth();
    for (DeviceId d : op.dst) bw = std::min(bw, link_bandwidth(cluster, op.src, d));
    busy[op.src] += static_cast<double>(op.bytes) / bw;
    plan.total_bytes += op.bytes * static_cast<Bytes>(op.dst.size());
  }
  for (const auto& kv : busy) plan.est_time = std::max(plan.est_time, kv.second);
  return plan;
}

std::string plan_to_json(const ReallocPlan& plan, const ModelSpec& model, const Placement& src,
                         const Placement& dst, const ClusterSpec& cluster) {
  std::ostringstream o;
  auto placement = [&](const Placement& p) {
    o << "{\"mesh\":\"" << mesh_to_string(p.mesh, cluster) << "\",\"dp\":" << p.strategy.dp
      << ",\"tp\":" << p.strategy.tp << ",\"pp\":" << p.strategy.pp
      << ",\"n_microbatches\":" << p.strategy.n_microbatches
      << ",\"qkv_layout\":" << static_cast<int>(p.qkv)
      << ",\"gate_up_layout\":" << static_cast<int>(p.gate_up) << ",\"kv_layout\":" << static_cast<int>(p.kv)
      << "}";
  };
  auto ops = [&](const std::vector<BroadcastOp>& list) {
    o << "[";
    for (size_t i = 0; i < list.size(); ++i) {
      const auto& op = list[i];
      o << (i ? "," : "") << "{\"src\":" << op.src << ",\"dst\":[";
      for (size_t k = 0; k < op.dst.size(); ++k) o << (k ? "," : "") << op.dst[k];
      o << "],\"layer_range\":[" << op.payload.layer_start << "," << op.payload.layer_end
        << "],\"slice_index\":" << op.payload.tp_rank
        << ",\"slice_count\":" << op.payload.tp_degree
        << ",\"replicated\":" << (op.payload.replicated ? "true" : "false")
        << (op.payload.part ? (op.payload.part == kPartKv ? ",\"part\":\"kv\"" : ",\"part\":\"no_kv\"") : "")
        << ",\"bytes\":" << op.bytes << "}";
    }
    o << "]";
  };
  char est[64];
  std::snprintf(est, sizeof(est), "%.17g", plan.est_time);
  o << "{\"schema\":1,\"model\":\"" << model.name << "\",\"src\":";
  placement(src);
  o << ",\"dst\":";
  placement(dst);
  o << ",\"total_bytes\":" << plan.total_bytes << ",\"est_time\":" << est << ",\"ops\":";
  ops(plan.ops);
  o << ",\"local_ops\":";
  ops(plan.local_ops);
  o << "}";
  return o.str();
}

namespace {

struct Rect {
  Count r0, r1, c0, c1;
  bool empty() const { return r0 >= r1 || c0 >= c1; }
};

Rect intersect(const Rect& a, const Rect& b) {
  return {std::max(a.r0, b.r0), std::min(a.r1, b.r1), std::max(a.c0, b.c0), std::min(a.c1, b.c1)};
}

// Blocks of a layout grouped by tensor id.
std::map<int, std::vector<const TensorBlock*>> by_tensor(const ShardLayout& lay) {
  std::map<int, std::vector<const TensorBlock*>> idx;
  for (const auto& b : lay.blocks) idx[b.tensor].push_back(&b);
  return idx;
}

Bytes block_offset(const TensorBlock& b, Count r, Count c, Bytes pb) {
  return b.offset + ((r - b.r0) * (b.c1 - b.c0) + (c - b.c0)) * pb;
}

}  // namespace

std::vector<LoweredOp> lower_plan(const ModelSpec& m, const Placement& src, const Placement& dst,
                                  const ClusterSpec& cluster, const ReallocPlan& plan) {
  const auto inv = tensor_inventory(m);
  const Bytes pb = m.param_bytes;
  std::vector<LoweredOp> out;
  std::map<OpKey, size_t> index;
  for (const auto* list : {&plan.ops, &plan.local_ops}) {
    for (const auto& op : *list) {
      const OpKey key = key_of(op.src, op.payload);
      auto it = index.find(key);
      if (it == index.end()) {
        it = index.emplace(key, out.size()).first;
        LoweredOp lo;
        lo.src = op.src;
        lo.payload = op.payload;
        lo.bytes = op.bytes;
        out.push_back(std::move(lo));
      }
      auto& dsts = out[it->second].dst;
      dsts.insert(dsts.end(), op.dst.begin(), op.dst.end());
    }
  }
  std::map<DeviceId, ShardLayout> s_lay, d_lay;
  for (auto& lo : out) {
    std::sort(lo.dst.begin(), lo.dst.end());
    const RankCoord r0 = rank_of(dst, cluster, lo.dst.front());
    for (DeviceId d : lo.dst) {
      const RankCoord rc = rank_of(dst, cluster, d);
      // Shards of one stage share their byte layout across TP ranks, so a
      // replicated payload may fan out to every TP rank, and so may a K/V
      // slice held by several ranks (replicated heads, G6); any other split
      // slice belongs to exactly one destination TP rank.
      const bool shared = lo.payload.replicated || lo.payload.part == kPartKv;
      if (rc.pp_rank != r0.pp_rank || (!shared && rc.tp_rank != r0.tp_rank))
        throw ValidationError("lower_plan: destinations of one op differ in geometry");
    }
    if (!s_lay.count(lo.src)) s_lay[lo.src] = shard_layout(m, src, cluster, lo.src);
    if (!d_lay.count(lo.dst.front())) d_lay[lo.dst.front()] = shard_layout(m, dst, cluster, lo.dst.front());
    if (lo.payload.part == kPartKv) {
      // the rectangles below are computed for dst.front() and stored at the
      // same offsets on every destination: their K/V blocks must coincide
      for (DeviceId d : lo.dst) {
        if (!d_lay.count(d)) d_lay[d] = shard_layout(m, dst, cluster, d);
        const auto& a = d_lay[lo.dst.front()].blocks;
        const auto& b = d_lay[d].blocks;
        bool same = a.size() == b.size();
        for (size_t i = 0; same && i < a.size(); ++i) {
          const int kind = inv[static_cast<size_t>(a[i].tensor)].kind;
          if (kind != kK && kind != kV) continue;
          same = a[i].tensor == b[i].tensor && a[i].r0 == b[i].r0 && a[i].r1 == b[i].r1 && a[i].offset == b[i].offset;
        }
        if (!same) throw ValidationError("lower_plan: K/V destinations of one op hold different blocks");
      }
    }
    const auto sidx = by_tensor(s_lay[lo.src]);
    const auto didx = by_tensor(d_lay[lo.dst.front()]);
    const ShardDescriptor& p = lo.payload;
    for (const auto& T : inv) {
      if (T.ext_layer < p.layer_start || T.ext_layer >= p.layer_end) continue;
      if (!in_payload(T, p.replicated, p.part)) continue;
      Rect want{0, T.rows, 0, T.cols};
      if (T.split == SplitKind::Rows) {
        want.r0 = p.tp_rank * T.rows / p.tp_degree;
        want.r1 = (p.tp_rank + 1) * T.rows / p.tp_degree;
      } else if (T.split == SplitKind::Cols) {
        want.c0 = p.tp_rank * T.cols / p.tp_degree;
        want.c1 = (p.tp_rank + 1) * T.cols / p.tp_degree;
      }
      const auto si = sidx.find(T.id);
      const auto di = didx.find(T.id);
      if (si == sidx.end() || di == didx.end())
        throw ValidationError("lower_plan: payload tensor missing from a shard layout");
      Count covered = 0;
      for (const TensorBlock* bs : si->second) {
        const Rect a = intersect(want, {bs->r0, bs->r1, bs->c0, bs->c1});
        if (a.empty()) continue;
        for (const TensorBlock* bd : di->second) {
          const Rect x = intersect(a, {bd->r0, bd->r1, bd->c0, bd->c1});
          if (x.empty()) continue;
          CopyRect cr;
          cr.src_off = block_offset(*bs, x.r0, x.c0, pb);
          cr.dst_off = block_offset(*bd, x.r0, x.c0, pb);
          cr.row_bytes = (x.c1 - x.c0) * pb;
          cr.src_pitch = (bs->c1 - bs->c0) * pb;
          cr.dst_pitch = (bd->c1 - bd->c0) * pb;
          cr.rows = x.r1 - x.r0;
          covered += (x.r1 - x.r0) * (x.c1 - x.c0);
          if (cr.rows > 1 && cr.src_pitch == cr.row_bytes && cr.dst_pitch == cr.row_bytes) {
            cr.row_bytes *= cr.rows;
            cr.rows = 1;
          }
          if (cr.rows == 1) cr.src_pitch = cr.dst_pitch = cr.row_bytes;
          // Coalesce with the previous rectangle when both sides continue it.
          if (!lo.rects.empty()) {
            CopyRect& prev = lo.rects.back();
            if (prev.rows == 1 && cr.rows == 1 && prev.src_off + prev.row_bytes == cr.src_off &&
                prev.dst_off + prev.row_bytes == cr.dst_off) {
              prev.row_bytes += cr.row_bytes;
              prev.src_pitch = prev.dst_pitch = prev.row_bytes;
              continue;
            }
          }
          lo.rects.push_back(cr);
        }
      }
      if (covered != (want.r1 - want.r0) * (want.c1 - want.c0))
        throw ValidationError("lower_plan: source/destination layouts do not cover the payload");
    }
    // Bounds: every rectangle lies inside both shards (compute-sanitizer is
    // unavailable on the GPU pool, so out-of-bounds copies are ruled out here).
    const Bytes s_bytes = s_lay[lo.src].bytes, d_bytes = d_lay[lo.dst.front()].bytes;
    for (const auto& r : lo.rects) {
      const Bytes s_end = r.src_off + (r.rows - 1) * r.src_pitch + r.row_bytes;
      const Bytes d_end = r.dst_off + (r.rows - 1) * r.dst_pitch + r.row_bytes;
      if (r.src_off < 0 || r.dst_off < 0 || r.rows < 1 || r.row_bytes < 1 || s_end > s_bytes || d_end > d_bytes)
        throw ValidationError("lower_plan: copy rectangle outside a shard");
    }
  }
  return out;
}

}  // namespace rlplan
