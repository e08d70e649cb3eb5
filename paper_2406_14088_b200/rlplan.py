"""Python mirror of the reference ``rlplan`` API, bound to librrealloc.so.

Names, fields, defaults and error behaviour follow the reference headers
(/root/reference/proj/include/rlplan/common.hpp, model_arith.hpp,
cluster.hpp) and the SPEC realloc module. Every call goes
through the C ABI (include/rr_realloc.h); nothing here re-implements the
planner.
"""
from __future__ import annotations

import ctypes
import json
import math
from dataclasses import dataclass, field, replace
from typing import Dict, List, Optional, Sequence, Tuple

from ._lib import (RrCluster, RrMesh, RrModel, RrOp, RrPlacement, ValidationError, check, lib)

__all__ = [
    "ValidationError", "ModelSpec", "ClusterSpec", "DeviceMesh", "ParallelStrategy", "Placement",
    "ShardDescriptor", "BroadcastOp", "ReallocPlan", "Phase", "param_count", "natural_param_count",
    "flops", "layer_flops_fwd", "kv_cache_bytes", "logits_bytes", "static_param_bytes",
    "validate_mesh", "enumerate_meshes", "overlap", "link_bandwidth", "local_bandwidth",
    "mesh_to_string", "mesh_from_string", "stage_layer_map", "validate_placement",
    "plan_param_realloc", "plan_data_transfer", "is_power_of_two", "ceil_div", "MODELS", "b200_cluster",
    "QKV_SEPARATE", "QKV_CONCAT", "QKV_GROUPED", "GATE_UP_SEPARATE", "GATE_UP_CONCAT", "KV_SPLIT",
    "KV_REPLICATE_HEADS", "PART_ALL", "PART_NO_KV", "PART_KV",
    "SPEC", "BALANCED",
]

QKV_SEPARATE, QKV_CONCAT, QKV_GROUPED = 0, 1, 2
# K/V when tp > kv heads (DESIGN.md §3 G6): rows split evenly, or whole heads replicated (Megatron/vLLM)
KV_SPLIT, KV_REPLICATE_HEADS = 0, 1
# ShardDescriptor.part: every TP-split tensor, all but k/v, k/v only (G6)
PART_ALL, PART_NO_KV, PART_KV = 0, 1, 2
GATE_UP_SEPARATE, GATE_UP_CONCAT = 0, 1
SPEC, BALANCED = 0, 1


def is_power_of_two(x: int) -> bool:  # reference common.hpp:17
    return x > 0 and (x & (x - 1)) == 0


def ceil_div(a: int, b: int) -> int:  # reference common.hpp:19
    return (a + b - 1) // b


@dataclass(frozen=True)
class ModelSpec:
    """reference model_arith.hpp:13-35."""
    name: str = ""
    hidden_size: int = 0
    intermediate_size: int = 0
    num_layers: int = 0
    num_attention_heads: int = 0
    num_kv_heads: int = 0
    vocab_size: int = 0
    max_position_embeddings: int = 0
    param_bytes: int = 2
    grad_bytes: int = 2
    optimizer_bytes_per_param: int = 12
    has_output_head: bool = True

    def head_dim(self) -> int:
        return self.hidden_size // self.num_attention_heads

    def validate(self) -> None:
        check(lib.rr_model_validate(ctypes.byref(self._c())))

    def _c(self) -> RrModel:
        return RrModel(self.name.encode(), self.hidden_size, self.intermediate_size, self.num_layers,
                       self.num_attention_heads, self.num_kv_heads, self.vocab_size,
                       self.max_position_embeddings, self.param_bytes, self.grad_bytes,
                       self.optimizer_bytes_per_param, 1 if self.has_output_head else 0)


@dataclass(frozen=True)
class ClusterSpec:
    """reference cluster.hpp:14-24."""
    n_nodes: int = 1
    gpus_per_node: int = 1
    mem_per_device: int = 0
    intra_node_bw: float = 0.0
    inter_node_bw: float = 0.0
    host_to_device_bw: float = 0.0

    def device_count(self) -> int:
        return self.n_nodes * self.gpus_per_node

    def validate(self) -> None:
        check(lib.rr_cluster_validate(ctypes.byref(self._c())))

    def _c(self) -> RrCluster:
        return RrCluster(self.n_nodes, self.gpus_per_node, self.mem_per_device, self.intra_node_bw,
                         self.inter_node_bw, self.host_to_device_bw)


@dataclass(frozen=True)
class DeviceMesh:
    """reference cluster.hpp:28-41."""
    node_offset: int = 0
    node_count: int = 1
    gpu_offset: int = 0
    gpu_count: int = 1

    def size(self) -> int:
        return self.node_count * self.gpu_count

    def devices(self, cluster: ClusterSpec) -> List[int]:
        buf = (ctypes.c_int32 * max(1, self.size()))()
        n = ctypes.c_int()
        check(lib.rr_mesh_devices(ctypes.byref(self._c()), ctypes.byref(cluster._c()), buf, len(buf),
                                  ctypes.byref(n)))
        return list(buf[: n.value])

    def first_device(self, cluster: ClusterSpec) -> int:
        return self.node_offset * cluster.gpus_per_node + self.gpu_offset

    def contains(self, cluster: ClusterSpec, d: int) -> bool:
        out = ctypes.c_int()
        check(lib.rr_mesh_contains(ctypes.byref(self._c()), ctypes.byref(cluster._c()), d, ctypes.byref(out)))
        return bool(out.value)

    def _c(self) -> RrMesh:
        return RrMesh(self.node_offset, self.node_count, self.gpu_offset, self.gpu_count)


@dataclass(frozen=True)
class ParallelStrategy:
    """SPEC.md:255-258."""
    dp: int = 1
    tp: int = 1
    pp: int = 1
    n_microbatches: int = 1


@dataclass(frozen=True)
class Placement:
    """(mesh, strategy) of one model function call plus its weight layout."""
    mesh: DeviceMesh
    strategy: ParallelStrategy
    qkv_layout: int = QKV_SEPARATE
    gate_up_layout: int = GATE_UP_SEPARATE
    kv_layout: int = KV_SPLIT

    def _c(self) -> RrPlacement:
        s = self.strategy
        return RrPlacement(self.mesh._c(), s.dp, s.tp, s.pp, s.n_microbatches, self.qkv_layout,
                           self.gate_up_layout, self.kv_layout)


@dataclass(frozen=True)
class ShardDescriptor:
    """SPEC.md:547-549 (layers -1 / L are the embedding / final norm + head)."""
    layer_start: int
    layer_end: int
    tp_rank: int
    tp_degree: int
    replicated: bool = False
    part: int = PART_ALL


@dataclass(frozen=True)
class BroadcastOp:
    """SPEC.md:550-552."""
    src: int
    dst: Tuple[int, ...]
    payload: ShardDescriptor
    bytes: int


class Phase:
    Forward = 0
    Backward = 1


# ---- model-arith (reference model_arith.hpp:37-72) -------------------------

def param_count(spec: ModelSpec, include_output_embedding: bool) -> int:
    out = ctypes.c_int64()
    check(lib.rr_param_count(ctypes.byref(spec._c()), int(include_output_embedding), ctypes.byref(out)))
    return out.value


def natural_param_count(spec: ModelSpec) -> int:
    out = ctypes.c_int64()
    check(lib.rr_natural_param_count(ctypes.byref(spec._c()), ctypes.byref(out)))
    return out.value


def flops(spec: ModelSpec, phase: int, tokens: int, context_len: int) -> float:
    out = ctypes.c_double()
    check(lib.rr_flops(ctypes.byref(spec._c()), int(phase), tokens, context_len, ctypes.byref(out)))
    return out.value


def layer_flops_fwd(spec: ModelSpec, tokens: int, context_len: int) -> float:
    out = ctypes.c_double()
    check(lib.rr_layer_flops_fwd(ctypes.byref(spec._c()), tokens, context_len, ctypes.byref(out)))
    return out.value


def kv_cache_bytes(spec: ModelSpec, batch: int, seq_len: int) -> int:
    out = ctypes.c_int64()
    check(lib.rr_kv_cache_bytes(ctypes.byref(spec._c()), batch, seq_len, ctypes.byref(out)))
    return out.value


def logits_bytes(vocab: int, batch: int, ctx_len: int, elem_bytes: int) -> int:
    out = ctypes.c_int64()
    check(lib.rr_logits_bytes(vocab, batch, ctx_len, elem_bytes, ctypes.byref(out)))
    return out.value


def static_param_bytes(spec: ModelSpec) -> Tuple[int, int, int]:
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    check(lib.rr_static_param_bytes(ctypes.byref(spec._c()), ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return a.value, b.value, c.value


# ---- cluster-topo (reference cluster.hpp:43-63) ----------------------------

def validate_mesh(mesh: DeviceMesh, cluster: ClusterSpec) -> None:
    check(lib.rr_validate_mesh(ctypes.byref(mesh._c()), ctypes.byref(cluster._c())))


def enumerate_meshes(cluster: ClusterSpec) -> List[DeviceMesh]:
    n = ctypes.c_int()
    cap = 64
    while True:
        buf = (RrMesh * cap)()
        st = lib.rr_enumerate_meshes(ctypes.byref(cluster._c()), buf, cap, ctypes.byref(n))
        if st == 6 and n.value > cap:  # RR_ERANGE
            cap = n.value
            continue
        check(st)
        return [DeviceMesh(m.node_offset, m.node_count, m.gpu_offset, m.gpu_count) for m in buf[: n.value]]


def overlap(a: DeviceMesh, b: DeviceMesh, cluster: ClusterSpec) -> bool:
    out = ctypes.c_int()
    check(lib.rr_overlap(ctypes.byref(a._c()), ctypes.byref(b._c()), ctypes.byref(cluster._c()), ctypes.byref(out)))
    return bool(out.value)


def link_bandwidth(cluster: ClusterSpec, a: int, b: int) -> float:
    out = ctypes.c_double()
    check(lib.rr_link_bandwidth(ctypes.byref(cluster._c()), a, b, ctypes.byref(out)))
    return out.value


def local_bandwidth() -> float:
    return math.inf


def mesh_to_string(mesh: DeviceMesh, cluster: ClusterSpec) -> str:
    buf = ctypes.create_string_buffer(128)
    need = ctypes.c_size_t()
    check(lib.rr_mesh_to_string(ctypes.byref(mesh._c()), ctypes.byref(cluster._c()), buf, 128, ctypes.byref(need)))
    return buf.value.decode()


def mesh_from_string(text: str, cluster: ClusterSpec) -> DeviceMesh:
    out = RrMesh()
    check(lib.rr_mesh_from_string(text.encode(), ctypes.byref(cluster._c()), ctypes.byref(out)))
    return DeviceMesh(out.node_offset, out.node_count, out.gpu_offset, out.gpu_count)


# ---- realloc ---------------------------------------------

def stage_layer_map(num_layers: int, pp: int) -> List[Tuple[int, int]]:
    n = max(pp, 1)
    starts, ends = (ctypes.c_int64 * n)(), (ctypes.c_int64 * n)()
    check(lib.rr_stage_layer_map(num_layers, pp, starts, ends))
    return [(starts[i], ends[i]) for i in range(pp)]


def validate_placement(model: ModelSpec, p: Placement, cluster: ClusterSpec) -> None:
    check(lib.rr_validate_placement(ctypes.byref(model._c()), ctypes.byref(p._c()), ctypes.byref(cluster._c())))


class ReallocPlan:
    """SPEC.md:553-557; owns the C plan (ops, lowering, layouts)."""

    def __init__(self, handle: int, model: ModelSpec, src: Placement, dst: Placement, cluster: ClusterSpec,
                 policy: int):
        self._h = ctypes.c_void_p(handle)
        self.model, self.src, self.dst, self.cluster, self.policy = model, src, dst, cluster, policy
        tb, et = ctypes.c_int64(), ctypes.c_double()
        check(lib.rr_plan_totals(self._h, ctypes.byref(tb), ctypes.byref(et)))
        self.total_bytes: int = tb.value
        self.est_time: float = et.value
        self.ops: List[BroadcastOp] = self._ops(0)
        self.local_ops: List[BroadcastOp] = self._ops(1)

    def _ops(self, local: int) -> List[BroadcastOp]:
        n = ctypes.c_int()
        check(lib.rr_plan_num_ops(self._h, local, ctypes.byref(n)))
        out = []
        for i in range(n.value):
            op = RrOp()
            check(lib.rr_plan_get_op(self._h, local, i, ctypes.byref(op)))
            p = op.payload
            out.append(BroadcastOp(op.src, tuple(op.dst[k] for k in range(op.n_dst)),
                                   ShardDescriptor(p.layer_start, p.layer_end, p.tp_rank, p.tp_degree,
                                                   bool(p.replicated), p.part), op.bytes))
        return out

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def to_json(self) -> dict:
        need = ctypes.c_size_t()
        lib.rr_plan_to_json(self._h, None, 0, ctypes.byref(need))
        buf = ctypes.create_string_buffer(need.value)
        check(lib.rr_plan_to_json(self._h, buf, need.value, ctypes.byref(need)))
        return json.loads(buf.value.decode())

    def shard_bytes(self, side: int, device: int) -> int:
        out = ctypes.c_int64()
        check(lib.rr_plan_shard_bytes(self._h, side, device, ctypes.byref(out)))
        return out.value

    def device_traffic(self, device: int) -> Tuple[int, int, int]:
        """(bytes in over links, bytes out over links, bytes copied locally)."""
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(lib.rr_plan_device_traffic(self._h, device, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    def num_rects(self) -> int:
        out = ctypes.c_int64()
        check(lib.rr_plan_num_rects(self._h, ctypes.byref(out)))
        return out.value

    def layout(self, side: int, device: int) -> List[Tuple[int, int, int, int, int, int]]:
        """Blocks (tensor, r0, r1, c0, c1, byte offset) of a device's shard."""
        n = ctypes.c_int64()
        lib.rr_plan_layout(self._h, side, device, None, 0, ctypes.byref(n))
        buf = (ctypes.c_int64 * max(1, 6 * n.value))()
        check(lib.rr_plan_layout(self._h, side, device, buf, n.value, ctypes.byref(n)))
        return [tuple(buf[6 * i: 6 * i + 6]) for i in range(n.value)]

    def lowered(self) -> List[Tuple[int, Tuple[int, ...], List[Tuple[int, int, int, int, int, int]]]]:
        """Merged ops lowered to copy rectangles: (src, dsts, [(src_off, dst_off,
        row_bytes, src_pitch, dst_pitch, rows), ...])."""
        n = ctypes.c_int()
        check(lib.rr_plan_num_lowered(self._h, ctypes.byref(n)))
        out = []
        for i in range(n.value):
            s, nd, nr = ctypes.c_int32(), ctypes.c_int(), ctypes.c_int64()
            dst = (ctypes.c_int32 * 64)()
            check(lib.rr_plan_get_lowered(self._h, i, ctypes.byref(s), dst, ctypes.byref(nd), None, 0,
                                          ctypes.byref(nr)))
            rects = (ctypes.c_int64 * max(1, 6 * nr.value))()
            check(lib.rr_plan_get_lowered(self._h, i, ctypes.byref(s), dst, ctypes.byref(nd), rects, nr.value,
                                          ctypes.byref(nr)))
            out.append((s.value, tuple(dst[: nd.value]),
                        [tuple(rects[6 * k: 6 * k + 6]) for k in range(nr.value)]))
        return out

    def work(self, local: Sequence[int], mode: int = 0, host_of: Optional[Sequence[int]] = None) -> Dict[str, int]:
        """Bytes an executor driving `local` would move (host only): phase 0
        (direct) and phase 1 (in-host fan-out) reads/writes, and bytes
        entering / leaving its host over links."""
        arr = (ctypes.c_int32 * max(1, len(local)))(*local)
        n = self.cluster.device_count()
        hosts = (ctypes.c_int32 * n)(*host_of) if host_of is not None else None
        out = (ctypes.c_int64 * 6)()
        check(lib.rr_plan_work(self._h, len(local), arr, hosts, mode, out))
        keys = ("read", "written", "fanout_read", "fanout_written", "wire_in", "wire_out")
        return dict(zip(keys, out))

    def ce_runs(self, local: Sequence[int], host_of: Optional[Sequence[int]] = None,
                min_run_bytes: int = 256 << 20) -> List[Tuple[int, int, int, int, int]]:
        """Copy-engine runs a push executor driving `local` would issue (host
        only): (src device, dst device, src offset, dst offset, bytes)."""
        arr = (ctypes.c_int32 * max(1, len(local)))(*local)
        n = self.cluster.device_count()
        hosts = (ctypes.c_int32 * n)(*host_of) if host_of is not None else None
        cnt = ctypes.c_int()
        check(lib.rr_plan_ce_runs(self._h, len(local), arr, hosts, min_run_bytes, None, 0, ctypes.byref(cnt)))
        out = (ctypes.c_int64 * (5 * max(1, cnt.value)))()
        check(lib.rr_plan_ce_runs(self._h, len(local), arr, hosts, min_run_bytes, out, cnt.value, ctypes.byref(cnt)))
        return [tuple(out[5 * i:5 * i + 5]) for i in range(cnt.value)]

    def ce_copies(self, local: Sequence[int], host_of: Optional[Sequence[int]] = None) -> List[Tuple[int, ...]]:
        """Copy-engine transport copies a push executor driving `local` would
        issue, in issue order (host only): (src device, dst device, src offset,
        dst offset, width, height, depth, src pitch, dst pitch, src slice
        stride, dst slice stride)."""
        arr = (ctypes.c_int32 * max(1, len(local)))(*local)
        n = self.cluster.device_count()
        hosts = (ctypes.c_int32 * n)(*host_of) if host_of is not None else None
        cnt = ctypes.c_int()
        check(lib.rr_plan_ce_copies(self._h, len(local), arr, hosts, None, 0, ctypes.byref(cnt)))
        out = (ctypes.c_int64 * (11 * max(1, cnt.value)))()
        check(lib.rr_plan_ce_copies(self._h, len(local), arr, hosts, out, cnt.value, ctypes.byref(cnt)))
        return [tuple(out[11 * i:11 * i + 11]) for i in range(cnt.value)]

    def ce_schedule(self, host_of: Sequence[int]) -> List[Tuple[int, int, float, float, bool, int]]:
        """The copy-engine transport schedule of every host (host only):
        (sender, receiver, simulated start s, end s, waits for another sender,
        bytes), each sender's transfers in issue order."""
        n = self.cluster.device_count()
        hosts = (ctypes.c_int32 * n)(*host_of)
        cnt = ctypes.c_int()
        check(lib.rr_plan_ce_schedule(self._h, hosts, None, 0, ctypes.byref(cnt)))
        out = (ctypes.c_double * (6 * max(1, cnt.value)))()
        check(lib.rr_plan_ce_schedule(self._h, hosts, out, cnt.value, ctypes.byref(cnt)))
        return [(int(out[6 * i]), int(out[6 * i + 1]), out[6 * i + 2], out[6 * i + 3], bool(out[6 * i + 4]),
                 int(out[6 * i + 5])) for i in range(cnt.value)]

    def devices(self, side: int) -> List[int]:
        p = self.src if side == 0 else self.dst
        return p.mesh.devices(self.cluster)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.rr_plan_destroy(h)
            self._h = ctypes.c_void_p(0)


def plan_data_transfer(producer: Placement, consumer: Placement, data_bytes_per_dp_shard: int,
                       cluster: ClusterSpec, policy: int = SPEC) -> ReallocPlan:
    """the realloc algorithm with TP and DP exchanged. Payloads
    are slices (tp_rank of tp_degree = lcm(dp)) of the data; the producer's
    outputs live on its last pipeline stage, every consumer device of a DP
    group needs that group's slices (DESIGN.md §3 G13)."""
    h = ctypes.c_void_p()
    check(lib.rr_plan_create_data(ctypes.byref(producer._c()), ctypes.byref(consumer._c()),
                                  ctypes.byref(cluster._c()), data_bytes_per_dp_shard, policy, ctypes.byref(h)))
    plan = ReallocPlan(h.value, None, producer, consumer, cluster, policy)
    plan.data_total = data_bytes_per_dp_shard * producer.strategy.dp
    return plan


def plan_param_realloc(model: ModelSpec, src: Placement, dst: Placement, cluster: ClusterSpec,
                       policy: int = SPEC) -> ReallocPlan:
    """SPEC.md:569-577. policy SPEC (lowest-index tie-break) or BALANCED."""
    h = ctypes.c_void_p()
    check(lib.rr_plan_create(ctypes.byref(model._c()), ctypes.byref(src._c()), ctypes.byref(dst._c()),
                             ctypes.byref(cluster._c()), policy, ctypes.byref(h)))
    return ReallocPlan(h.value, model, src, dst, cluster, policy)


# ---- presets ------------------------------------------------------------------

def _llama(name, h, i, L, heads, kv, vocab=128256, head=True):
    return ModelSpec(name=name, hidden_size=h, intermediate_size=i, num_layers=L, num_attention_heads=heads,
                     num_kv_heads=kv, vocab_size=vocab, max_position_embeddings=8192, has_output_head=head)


# Appendix-A shapes; "tiny" is BASELINE.json configs[0]
# (4 layers, hidden 256) with the remaining dims chosen in SURVEY.md §8 a3;
# "spec_tiny" is the SPEC.md:47 tiny spec.
MODELS: Dict[str, ModelSpec] = {
    "tiny": _llama("tiny", 256, 688, 4, 4, 2, vocab=1024),
    "spec_tiny": ModelSpec(name="spec_tiny", hidden_size=4, intermediate_size=8, num_layers=1,
                           num_attention_heads=2, num_kv_heads=1, vocab_size=10, max_position_embeddings=16),
    "llama7b": _llama("llama7b", 4096, 14336, 32, 32, 8),
    "llama13b": _llama("llama13b", 5120, 13824, 40, 40, 40),
    "llama34b_critic": _llama("llama34b_critic", 8192, 22016, 48, 64, 8, head=False),
    "llama34b": _llama("llama34b", 8192, 22016, 48, 64, 8),
    "llama70b": _llama("llama70b", 8192, 28672, 80, 64, 8),
}


def b200_cluster(gpus: int = 8, nodes: int = 1) -> ClusterSpec:
    """One HGX B200 box: NVSwitch gives every peer 900 GB/s per direction."""
    return ClusterSpec(n_nodes=nodes, gpus_per_node=gpus, mem_per_device=183359 * 2**20,
                       intra_node_bw=900e9, inter_node_bw=50e9, host_to_device_bw=55e9)
