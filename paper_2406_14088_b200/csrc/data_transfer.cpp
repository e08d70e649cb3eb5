// Inter-call data transfer: the parameter
// reallocation algorithm with the roles of TP and DP exchanged. Data of one
// function call is split into disjoint DP partitions and replicated across TP;
// the consumer re-slices at lcm(dp_producer, dp_consumer) granularity.
#include <algorithm>
#include <map>
#include <tuple>

#include "rlplan/realloc.hpp"

namespace rlplan {

namespace {

void validate_strategy(const Placement& p, const ClusterSpec& cluster, const char* who) {
  validate_mesh(p.mesh, cluster);
  const ParallelStrategy& s = p.strategy;
  auto need = [&](bool ok, const char* why) {
    if (!ok) throw ValidationError(std::string("plan_data_transfer: ") + who + " " + why);
  };
  need(s.dp >= 1 && s.tp >= 1 && s.pp >= 1, "dp, tp, pp must be >= 1");
  need(s.n_microbatches >= 1, "n_microbatches must be >= 1");
  need(static_cast<Count>(s.dp) * s.tp * s.pp == p.mesh.size(), "dp*tp*pp must equal the mesh size");
}

}  // namespace

ReallocPlan plan_data_transfer(const Placement& prod, const Placement& cons, Bytes data_bytes_per_dp_shard,
                               const ClusterSpec& cluster, SourcePolicy policy) {
  cluster.validate();
  validate_strategy(prod, cluster, "producer");
  validate_strategy(cons, cluster, "consumer");
  const int dp1 = prod.strategy.dp, dp2 = cons.strategy.dp;
  const int G = static_cast<int>(lcm_count(dp1, dp2));
  if (data_bytes_per_dp_shard <= 0) throw ValidationError("plan_data_transfer: data bytes must be positive");
  const Bytes total = data_bytes_per_dp_shard * dp1;
  if (total % (2 * G))
    throw ValidationError("plan_data_transfer: data does not split into lcm(dp) equal bf16 slices");
  const Bytes slice = total / G;

  ReallocPlan plan;
  using Key = std::tuple<DeviceId, int>;
  std::map<Key, size_t> remote, local;
  std::map<DeviceId, Bytes> egress;
  for (DeviceId d : cons.mesh.devices(cluster)) {  // ascending = (pp, dp, tp) rank order
    const RankCoord rc = rank_of(cons, cluster, d);
    for (int k = rc.dp_rank * (G / dp2); k < (rc.dp_rank + 1) * (G / dp2); ++k) {
      std::vector<DeviceId> holders;  // every (pp, tp) replica of the producer's DP slice
      for (int s = 0; s < prod.strategy.pp; ++s)
        for (int t = 0; t < prod.strategy.tp; ++t) holders.push_back(device_at(prod, cluster, s, k / (G / dp1), t));
      std::sort(holders.begin(), holders.end());
      DeviceId pick = -1;
      if (std::find(holders.begin(), holders.end(), d) != holders.end()) {
        pick = d;
      } else {
        double best = -1;
        for (DeviceId h : holders) best = std::max(best, link_bandwidth(cluster, h, d));
        for (DeviceId h : holders) {
          if (link_bandwidth(cluster, h, d) != best) continue;
          if (pick < 0 || (policy == SourcePolicy::Balanced && egress[h] < egress[pick])) pick = h;
          if (policy == SourcePolicy::Spec) break;
        }
        egress[pick] += slice;
      }
      auto& index = pick == d ? local : remote;
      auto& list = pick == d ? plan.local_ops : plan.ops;
      auto it = index.find({pick, k});
      if (it == index.end()) {
        it = index.emplace(Key{pick, k}, list.size()).first;
        list.push_back(BroadcastOp{pick, {}, ShardDescriptor{0, 0, k, G, false}, slice});
      }
      list[it->second].dst.push_back(d);
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

ShardLayout data_layout(const Placement& p, const ClusterSpec& cluster, DeviceId d, Bytes total_bytes,
                        bool producer) {
  ShardLayout lay;
  const RankCoord rc = rank_of(p, cluster, d);
  if (!rc.valid()) return lay;
  (void)producer;  // producer and consumer devices both hold their DP group's data
  const Count elems = total_bytes / 2;
  const Count per = elems / p.strategy.dp;
  lay.blocks.push_back({kDataTensor, 0, 1, rc.dp_rank * per, (rc.dp_rank + 1) * per, 0});
  lay.bytes = (per * 2 + 255) / 256 * 256;
  return lay;
}

std::vector<LoweredOp> lower_data_plan(const Placement& prod, const Placement& cons, const ClusterSpec& cluster,
                                       Bytes total_bytes, const ReallocPlan& plan) {
  const Count elems = total_bytes / 2;
  std::vector<LoweredOp> out;
  std::map<std::tuple<DeviceId, int>, size_t> index;
  for (const auto* list : {&plan.ops, &plan.local_ops}) {
    for (const auto& op : *list) {
      auto key = std::make_tuple(op.src, op.payload.tp_rank);
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
  for (auto& lo : out) {
    std::sort(lo.dst.begin(), lo.dst.end());
    const Count s0 = lo.payload.tp_rank * elems / lo.payload.tp_degree;
    const Count s1 = (lo.payload.tp_rank + 1) * elems / lo.payload.tp_degree;
    const ShardLayout src = data_layout(prod, cluster, lo.src, total_bytes, true);
    const ShardLayout dst = data_layout(cons, cluster, lo.dst.front(), total_bytes, false);
    const TensorBlock& bs = src.blocks.at(0);
    const TensorBlock& bd = dst.blocks.at(0);
    for (DeviceId d : lo.dst)  // one DP group: identical element ranges
      if (data_layout(cons, cluster, d, total_bytes, false).blocks.at(0).c0 != bd.c0)
        throw ValidationError("lower_data_plan: destinations of one op differ in geometry");
    if (s0 < bs.c0 || s1 > bs.c1 || s0 < bd.c0 || s1 > bd.c1 || (s1 - bs.c0) * 2 > src.bytes ||
        (s1 - bd.c0) * 2 > dst.bytes)
      throw ValidationError("lower_data_plan: slice outside a shard");
    CopyRect r;
    r.src_off = (s0 - bs.c0) * 2;
    r.dst_off = (s0 - bd.c0) * 2;
    r.row_bytes = r.src_pitch = r.dst_pitch = (s1 - s0) * 2;
    r.rows = 1;
    lo.rects.push_back(r);
  }
  return out;
}

}  // namespace rlplan
