// Parameter reallocation: plan types, stage map, planner, layout contract and
// lowering to 2D copy rectangles.
//
// The reference declares this module only in SPEC.md:541-611 (types
// SPEC.md:546-557, stage_layer_map SPEC.md:560-568, plan_param_realloc
// SPEC.md:569-577, design decisions SPEC.md:594-598) and describes the
// algorithm in PAPER.md:500 and PAPER.md:514-515. Names follow the SPEC.
// Everything the SPEC leaves open (rank order, non-layer tensors, TP split
// kinds, fused layouts, byte layout of a shard) is pinned by the layout
// contract in DESIGN.md §3 and implemented by shard_layout() below.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "rlplan/cluster.hpp"
#include "rlplan/common.hpp"
#include "rlplan/model_arith.hpp"

namespace rlplan {

// 3D strategy of one placement. dp*tp*pp must equal the
// mesh size.
struct ParallelStrategy {
  int dp = 1;
  int tp = 1;
  int pp = 1;
  int n_microbatches = 1;
  bool operator==(const ParallelStrategy&) const = default;
};

// How a placement stores attention/MLP input projections (DESIGN.md §3 G4).
//   Separate: q, k, v as three tensors.
//   Concat:   one fused tensor per TP rank, rows [Q_r; K_r; V_r] (vLLM/HF).
//   Grouped:  Megatron fused QKV, rows grouped per KV head:
//             for each local KV group g: [q heads of g; k_g; v_g].
enum class QkvLayout : int { Separate = 0, Concat = 1, Grouped = 2 };
//   Separate: gate, up as two tensors.  Concat: rows [G_r; U_r].
enum class GateUpLayout : int { Separate = 0, Concat = 1 };
// K/V weights when tp exceeds the KV heads (DESIGN.md §3 G6).
//   Split:          k/v rows split evenly over tp like every row-split tensor
//                   (the reference's arithmetic).
//   ReplicateHeads: Megatron / vLLM: tp rank r holds whole KV head
//                   floor(r * kv_heads / tp); needs tp % kv_heads == 0.
//   Both are the same layout when tp <= kv_heads.
enum class KvLayout : int { Split = 0, ReplicateHeads = 1 };

struct Placement {
  DeviceMesh mesh;
  ParallelStrategy strategy;
  QkvLayout qkv = QkvLayout::Separate;
  GateUpLayout gate_up = GateUpLayout::Separate;
  KvLayout kv = KvLayout::Split;
};

// Number of distinct K/V slices a placement's TP ranks hold: kv_heads under
// ReplicateHeads with tp > kv_heads, else tp. Rank r holds slice
// floor(r * kv_degree / tp).
int kv_degree(const ModelSpec& model, const Placement& p);

// ValidationError unless the strategy fits the mesh and model: dp,tp,pp >= 1,
// dp*tp*pp == mesh size, pp <= num_layers, tp a power of two dividing the
// attention heads, and every TP-split dimension divisible by tp.
void validate_placement(const ModelSpec& model, const Placement& p, const ClusterSpec& cluster);

// Coordinates of a device inside a placement. Rank order over the mesh's
// ascending devices (DESIGN.md §3 G1): dev = devices[(pp*dp + dp_r)*tp + tp_r].
struct RankCoord {
  int pp_rank = -1;
  int dp_rank = -1;
  int tp_rank = -1;
  bool valid() const { return pp_rank >= 0; }
};
RankCoord rank_of(const Placement& p, const ClusterSpec& cluster, DeviceId d);
DeviceId device_at(const Placement& p, const ClusterSpec& cluster, int pp_rank, int dp_rank,
                   int tp_rank);

// Payload of a BroadcastOp. Layers are "extended" indices:
// -1 is the input embedding (held by stage 0), num_layers is the final norm
// plus the output head (held by the last stage), 0..L-1 are decoder layers
// (DESIGN.md §3 G2). A split payload is slice tp_rank of tp_degree =
// lcm(tp_src, tp_dst) of every TP-split tensor in the range;
// tp_degree == 1 with `replicated` set carries the replicated tensors
// (norms, scalar value head) of the range (G5).
//
// `part` separates K/V when a placement replicates KV heads (G6): a plan in
// which either side has kv_degree != tp carries split payloads without k/v
// (part 1) and K/V payloads (part 2: slice tp_rank of tp_degree =
// lcm(kv_degree_src, kv_degree_dst) of every k and v in the range). All
// other plans use part 0 (every TP-split tensor).
enum PayloadPart : int { kPartAll = 0, kPartNoKv = 1, kPartKv = 2 };

struct ShardDescriptor {
  Count layer_start = 0;
  Count layer_end = 0;
  int tp_rank = 0;
  int tp_degree = 1;
  bool replicated = false;
  int part = kPartAll;
  bool operator==(const ShardDescriptor&) const = default;
};

// One source broadcasting one payload to a set of destinations.
// `bytes` is the payload size; every destination receives all of it.
struct BroadcastOp {
  DeviceId src = -1;
  std::vector<DeviceId> dst;
  ShardDescriptor payload;
  Bytes bytes = 0;
};

// SPEC.md:553-557. `ops` carries only transfers that cross a link; payloads a
// destination already holds itself are listed in `local_ops` (src == dst[0],
// no wire bytes) so that an executor also knows which local relayout copies
// to perform. total_bytes = sum over ops of bytes * |dst| (bytes delivered
// over links); est_time = max over sources of sum(bytes / bandwidth)
// (SPEC.md:572).
struct ReallocPlan {
  std::vector<BroadcastOp> ops;
  Bytes total_bytes = 0;
  Seconds est_time = 0;
  std::vector<BroadcastOp> local_ops;
};

// Greedy source choice among equal-cost holders (DESIGN.md §3 G7).
//   Spec:     lowest device index, used for plan parity.
//   Balanced: least egress bytes assigned so far, then lowest index; same
//             bytes, spreads sender load when sources are DP replicas.
enum class SourcePolicy : int { Spec = 0, Balanced = 1 };

// Contiguous stages; the first (L mod pp) stages get ceil(L/pp) layers
// (SPEC.md:560-568). ValidationError if pp < 1 or pp > num_layers.
std::vector<std::pair<Count, Count>> stage_layer_map(Count num_layers, int pp);

// outer loop over stage pairs with common layers, inner
// loop over destination devices and required slices, cheapest holder wins
// (self > same node > other node), destinations sharing (src, payload) are
// grouped into one op.
ReallocPlan plan_param_realloc(const ModelSpec& model, const Placement& src, const Placement& dst,
                               const ClusterSpec& cluster,
                               SourcePolicy policy = SourcePolicy::Spec);

// data produced by one function call and consumed by the
// next. "Model function calls produce disjoint data partitions along the DP
// dimension, while replicating the data along the TP dimension":
// the same greedy broadcast algorithm with TP and DP exchanged. Payloads
// are slice tp_rank of tp_degree = lcm(dp_producer, dp_consumer) of the data
// (layer range [0, 0)). PP, like TP, is a replica axis for data: every
// device of a DP group holds (producer) or needs (consumer) that group's
// data, so identical placements give an empty plan (DESIGN.md
// §3 G13). ValidationError on invalid placements or when the data does not
// split into lcm(dp) equal 2-byte-aligned slices.
ReallocPlan plan_data_transfer(const Placement& producer, const Placement& consumer,
                               Bytes data_bytes_per_dp_shard, const ClusterSpec& cluster,
                               SourcePolicy policy = SourcePolicy::Spec);

// Bytes of one payload.
Bytes payload_bytes(const ModelSpec& model, const ShardDescriptor& payload);

// Plan file: op list with src, dst set,
// layer range, slice index, bytes.
std::string plan_to_json(const ReallocPlan& plan, const ModelSpec& model, const Placement& src,
                         const Placement& dst, const ClusterSpec& cluster);

// ---------------------------------------------------------------------------
// Layout contract: logical tensors and per-device shard bytes.
// ---------------------------------------------------------------------------

enum class SplitKind : int { Rows = 0, Cols = 1, Replicated = 2 };

// Logical (unsharded) weight, row-major [rows, cols] as stored [out, in].
struct LogicalTensor {
  int id = 0;             // canonical index, see tensor_inventory()
  Count ext_layer = 0;    // extended layer (-1 embed, L final)
  int kind = 0;           // TensorKind value
  Count rows = 0;
  Count cols = 0;
  SplitKind split = SplitKind::Replicated;
};

enum TensorKind : int {
  kEmbed = 0,
  kLn1 = 1,
  kQ = 2,
  kK = 3,
  kV = 4,
  kO = 5,
  kLn2 = 6,
  kGate = 7,
  kUp = 8,
  kDown = 9,
  kFinalNorm = 10,
  kHead = 11,   // vocab output head [V, h]
  kVHead = 12,  // scalar value head [1, h]
};

// Canonical tensor list: id 0 embed; layer l tensors 1+9l .. 9+9l in order
// ln1,q,k,v,o,ln2,gate,up,down; then final norm (1+9L) and head (2+9L).
// Sum of rows*cols == natural_param_count(model).
std::vector<LogicalTensor> tensor_inventory(const ModelSpec& model);

// A rectangle of one logical tensor stored row-major (pitch = c1 - c0
// elements) at byte offset `offset` of a device's shard buffer.
struct TensorBlock {
  int tensor = 0;
  Count r0 = 0, r1 = 0, c0 = 0, c1 = 0;
  Bytes offset = 0;
};

// Every block a device holds under a placement, in buffer order. Tensor
// entries start on 256-byte boundaries; the blocks of one fused entry are
// packed back to back.
struct ShardLayout {
  std::vector<TensorBlock> blocks;
  Bytes bytes = 0;
};
ShardLayout shard_layout(const ModelSpec& model, const Placement& p, const ClusterSpec& cluster,
                         DeviceId d);

// ---------------------------------------------------------------------------
// Lowering: plan -> per-op 2D copy rectangles shared by all of the op's
// destinations (every destination of an op has the same (stage, tp_rank),
// hence the same local geometry).
// ---------------------------------------------------------------------------

struct CopyRect {
  Bytes src_off = 0;
  Bytes dst_off = 0;
  Bytes row_bytes = 0;
  Bytes src_pitch = 0;
  Bytes dst_pitch = 0;
  Count rows = 0;
};

struct LoweredOp {
  DeviceId src = -1;
  std::vector<DeviceId> dst;  // includes src itself when it is also a destination
  ShardDescriptor payload;
  std::vector<CopyRect> rects;
  Bytes bytes = 0;            // payload bytes (per destination)
};

// ops and local_ops merged per (src, payload), then lowered.
std::vector<LoweredOp> lower_plan(const ModelSpec& model, const Placement& src,
                                  const Placement& dst, const ClusterSpec& cluster,
                                  const ReallocPlan& plan);

// ---------------------------------------------------------------------------
// Inter-call data (plan_data_transfer) layout and lowering.
// ---------------------------------------------------------------------------

// Tensor id of the (1-D, bf16-element) data a data-transfer plan moves.
constexpr int kDataTensor = 0x7fff0000;

// Data held (producer) or needed (consumer) by a device: its DP group's
// elements, one block [0,1) x [first, last) of kDataTensor at offset 0.
ShardLayout data_layout(const Placement& p, const ClusterSpec& cluster, DeviceId d, Bytes total_bytes,
                        bool producer);

// Data-transfer ops lowered to 1-D copy rectangles.
std::vector<LoweredOp> lower_data_plan(const Placement& producer, const Placement& consumer,
                                       const ClusterSpec& cluster, Bytes total_bytes, const ReallocPlan& plan);

}  // namespace rlplan
