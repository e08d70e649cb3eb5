// Layout contract: tensor inventory, placement validation, rank order and
// per-device shard layout (the reference leaves all of this
// open — SURVEY.md Appendix A G1-G10).
//
// The tensor set is exactly the one summed by reference
// proj/src/model_arith.cpp:28-46 (q,o h*h; k,v h*head_dim*kv; gate,up,down
// h*i; two norms; embedding, final norm, vocab head or scalar head).
#include <algorithm>

#include "rlplan/realloc.hpp"

namespace rlplan {

namespace {

constexpr Bytes kEntryAlign = 256;

Bytes align_up(Bytes v, Bytes a) { return (v + a - 1) / a * a; }

}  // namespace

std::vector<LogicalTensor> tensor_inventory(const ModelSpec& m) {
  m.validate();
  const Count h = m.hidden_size, L = m.num_layers;
  const Count q_rows = m.num_attention_heads * m.head_dim();
  const Count kv_rows = m.num_kv_heads * m.head_dim();
  const Count ffn = m.intermediate_size;
  std::vector<LogicalTensor> out;
  out.reserve(static_cast<size_t>(3 + 9 * L));
  auto add = [&](Count layer, int kind, Count rows, Count cols, SplitKind split) {
    out.push_back({static_cast<int>(out.size()), layer, kind, rows, cols, split});
  };
  add(-1, kEmbed, m.vocab_size, h, SplitKind::Rows);
  for (Count l = 0; l < L; ++l) {
    add(l, kLn1, 1, h, SplitKind::Replicated);
    add(l, kQ, q_rows, h, SplitKind::Rows);
    add(l, kK, kv_rows, h, SplitKind::Rows);
    add(l, kV, kv_rows, h, SplitKind::Rows);
    add(l, kO, h, q_rows, SplitKind::Cols);
    add(l, kLn2, 1, h, SplitKind::Replicated);
    add(l, kGate, ffn, h, SplitKind::Rows);
    add(l, kUp, ffn, h, SplitKind::Rows);
    add(l, kDown, h, ffn, SplitKind::Cols);
  }
  add(L, kFinalNorm, 1, h, SplitKind::Replicated);
  if (m.has_output_head)
    add(L, kHead, m.vocab_size, h, SplitKind::Rows);
  else
    add(L, kVHead, 1, h, SplitKind::Replicated);
  return out;
}

void validate_placement(const ModelSpec& m, const Placement& p, const ClusterSpec& cluster) {
  m.validate();
  validate_mesh(p.mesh, cluster);
  const ParallelStrategy& s = p.strategy;
  auto need = [](bool ok, const std::string& why) {
    if (!ok) throw ValidationError("Placement: " + why);
  };
  need(s.dp >= 1 && s.tp >= 1 && s.pp >= 1, "dp, tp, pp must be >= 1");
  need(s.n_microbatches >= 1, "n_microbatches must be >= 1");
  need(static_cast<Count>(s.dp) * s.tp * s.pp == p.mesh.size(),
       "dp*tp*pp must equal the mesh size");
  need(s.pp <= m.num_layers, "pp must not exceed num_layers");
  need(is_power_of_two(s.tp), "tp must be a power of two");
  need(m.num_attention_heads % s.tp == 0, "tp must divide num_attention_heads");
  const bool kv_heads = p.kv == KvLayout::ReplicateHeads && s.tp > m.num_kv_heads;
  for (const auto& t : tensor_inventory(m)) {
    if (kv_heads && (t.kind == kK || t.kind == kV)) continue;  // whole heads, checked below
    if (t.split == SplitKind::Rows) need(t.rows % s.tp == 0, "tp must divide every row-split dimension");
    if (t.split == SplitKind::Cols) need(t.cols % s.tp == 0, "tp must divide every column-split dimension");
  }
  const int q = static_cast<int>(p.qkv), g = static_cast<int>(p.gate_up);
  need(q >= 0 && q <= 2, "unknown qkv layout");
  need(g >= 0 && g <= 1, "unknown gate_up layout");
  if (p.qkv == QkvLayout::Grouped)
    need(m.num_kv_heads % s.tp == 0, "grouped QKV layout needs tp to divide num_kv_heads");
  const int kv = static_cast<int>(p.kv);
  need(kv >= 0 && kv <= 1, "unknown kv layout");
  if (p.kv == KvLayout::ReplicateHeads && s.tp > m.num_kv_heads)
    need(s.tp % m.num_kv_heads == 0, "replicated KV heads need tp to be a multiple of num_kv_heads");
}

int kv_degree(const ModelSpec& m, const Placement& p) {
  const int tp = p.strategy.tp;
  if (p.kv == KvLayout::ReplicateHeads && tp > m.num_kv_heads) return static_cast<int>(m.num_kv_heads);
  return tp;
}

RankCoord rank_of(const Placement& p, const ClusterSpec& cluster, DeviceId d) {
  RankCoord rc;
  if (!p.mesh.contains(cluster, d)) return rc;
  const auto devs = p.mesh.devices(cluster);
  const auto it = std::find(devs.begin(), devs.end(), d);
  if (it == devs.end()) return rc;
  const int idx = static_cast<int>(it - devs.begin());
  const ParallelStrategy& s = p.strategy;
  rc.tp_rank = idx % s.tp;
  rc.dp_rank = (idx / s.tp) % s.dp;
  rc.pp_rank = idx / (s.tp * s.dp);
  return rc;
}

DeviceId device_at(const Placement& p, const ClusterSpec& cluster, int pp_rank, int dp_rank,
                   int tp_rank) {
  const ParallelStrategy& s = p.strategy;
  const auto devs = p.mesh.devices(cluster);
  return devs[static_cast<size_t>((pp_rank * s.dp + dp_rank) * s.tp + tp_rank)];
}

ShardLayout shard_layout(const ModelSpec& m, const Placement& p, const ClusterSpec& cluster,
                         DeviceId d) {
  ShardLayout lay;
  const RankCoord rc = rank_of(p, cluster, d);
  if (!rc.valid()) return lay;
  const auto inv = tensor_inventory(m);
  const auto stages = stage_layer_map(m.num_layers, p.strategy.pp);
  const Count L = m.num_layers;
  const int t = p.strategy.tp, r = rc.tp_rank;
  const int e = kv_degree(m, p), kv_slice = r * e / t;  // K/V slice this rank holds (G6)
  const Bytes pb = m.param_bytes;
  Bytes cursor = 0;

  // Append the block [r0,r1)x[c0,c1) of tensor `id` at the cursor.
  auto put = [&](int id, Count r0, Count r1, Count c0, Count c1) {
    lay.blocks.push_back({id, r0, r1, c0, c1, cursor});
    cursor += (r1 - r0) * (c1 - c0) * pb;
  };
  // This rank's part of a tensor per its split kind.
  auto put_part = [&](int id) {
    const LogicalTensor& T = inv[static_cast<size_t>(id)];
    if (T.kind == kK || T.kind == kV) {
      put(id, kv_slice * T.rows / e, (kv_slice + 1) * T.rows / e, 0, T.cols);
      return;
    }
    switch (T.split) {
      case SplitKind::Rows: put(id, r * T.rows / t, (r + 1) * T.rows / t, 0, T.cols); break;
      case SplitKind::Cols: put(id, 0, T.rows, r * T.cols / t, (r + 1) * T.cols / t); break;
      case SplitKind::Replicated: put(id, 0, T.rows, 0, T.cols); break;
    }
  };
  auto begin_entry = [&]() { cursor = align_up(cursor, kEntryAlign); };

  const Count lo = stages[static_cast<size_t>(rc.pp_rank)].first - (rc.pp_rank == 0 ? 1 : 0);
  const Count hi = stages[static_cast<size_t>(rc.pp_rank)].second + (rc.pp_rank == p.strategy.pp - 1 ? 1 : 0);
  for (Count e = lo; e < hi; ++e) {
    if (e == -1) {
      begin_entry();
      put_part(0);
      continue;
    }
    if (e == L) {
      const int base = static_cast<int>(1 + 9 * L);
      begin_entry();
      put_part(base);
      begin_entry();
      put_part(base + 1);
      continue;
    }
    const int base = static_cast<int>(1 + 9 * e);
    const int ln1 = base, q = base + 1, k = base + 2, v = base + 3, o = base + 4, ln2 = base + 5,
              gate = base + 6, up = base + 7, down = base + 8;
    begin_entry();
    put_part(ln1);
    switch (p.qkv) {
      case QkvLayout::Separate:
        for (int id : {q, k, v}) {
          begin_entry();
          put_part(id);
        }
        break;
      case QkvLayout::Concat:
        begin_entry();
        for (int id : {q, k, v}) put_part(id);
        break;
      case QkvLayout::Grouped: {
        begin_entry();
        const Count hd = m.head_dim(), h = m.hidden_size;
        const Count groups = m.num_kv_heads, per_rank = groups / t;
        const Count q_per_group = m.num_attention_heads / groups * hd;
        for (Count g = r * per_rank; g < (r + 1) * per_rank; ++g) {
          put(q, g * q_per_group, (g + 1) * q_per_group, 0, h);
          put(k, g * hd, (g + 1) * hd, 0, h);
          put(v, g * hd, (g + 1) * hd, 0, h);
        }
        break;
      }
    }
    begin_entry();
    put_part(o);
    begin_entry();
    put_part(ln2);
    if (p.gate_up == GateUpLayout::Concat) {
      begin_entry();
      put_part(gate);
      put_part(up);
    } else {
      begin_entry();
      put_part(gate);
      begin_entry();
      put_part(up);
    }
    begin_entry();
    put_part(down);
  }
  lay.bytes = align_up(cursor, kEntryAlign);
  return lay;
}

}  // namespace rlplan
