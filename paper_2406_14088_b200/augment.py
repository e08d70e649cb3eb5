"""The simulator's ``augment`` step for this path, priced
with the measured B200 cost model.

The reference's simulator inserts extra nodes into an RLHF dataflow graph
for a given execution plan (Fig. 5): a
``param_realloc`` node wherever a model's consecutive calls run under
different (mesh, strategy), a ``data_transfer`` node on every data edge
whose producer and consumer placements differ, and ``offload`` / ``onload``
nodes for models flagged to park their parameters in host memory between
calls. SPEC prices them at ``bytes / bandwidth``
(SPEC.md:423). Here every inserted node carries that SPEC
estimate next to the time the B200 executor takes for the same plan
(``costmodel``), and the plan itself, so a simulator can use either.

The workflow DAG builders and the simulation proper (SPEC.md:175-248,
SPEC.md:429-462) are out of scope; callers pass the
calls of one iteration in execution order.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from . import costmodel
from .rlplan import (BALANCED, ClusterSpec, ModelSpec, Placement, ReallocPlan, plan_data_transfer,
                     plan_param_realloc)


@dataclass(frozen=True)
class Call:
    """One model function call of the workflow (SPEC.md:175-248 nodes) with
    its plan assignment (mesh, strategy, offload flag)."""
    name: str
    model: str                 # model handle, e.g. "actor", "critic"
    placement: Placement
    offload: bool = False      # park this model's parameters in host memory after the call


@dataclass(frozen=True)
class DataEdge:
    """Producer -> consumer data dependency; the producer's output is
    DP-partitioned, ``bytes_per_dp_shard`` per DP rank."""
    producer: str
    consumer: str
    bytes_per_dp_shard: int


@dataclass
class InsertedNode:
    kind: str                              # param_realloc | data_transfer | offload | onload
    between: Tuple[str, str]               # (after call, before call); offload/onload: (call, next call)
    model: Optional[str]
    bytes: int                             # bytes moved (plan total_bytes; per-GPU bytes for offload/onload)
    spec_seconds: float                    # SPEC.md:423 / SPEC.md:572 estimate
    b200_seconds: float                    # measured B200 cost model
    plan: Optional[ReallocPlan] = field(default=None, repr=False)


def _grid(p: Placement) -> tuple:
    """What decides who holds which bytes (n_microbatches does not)."""
    s = p.strategy
    return (p.mesh, s.dp, s.tp, s.pp)


def _same(a: Placement, b: Placement) -> bool:
    return _grid(a) == _grid(b) and a.qkv_layout == b.qkv_layout and a.gate_up_layout == b.gate_up_layout


def _shard_max(plan: ReallocPlan, side: int) -> int:
    return max((plan.shard_bytes(side, d) for d in plan.devices(side)), default=0)


def augment(calls: Sequence[Call], edges: Sequence[DataEdge], models: Dict[str, ModelSpec],
            cluster: ClusterSpec, cyclic: bool = True, policy: int = BALANCED,
            profile: costmodel.B200Profile = costmodel.B200Profile()) -> List[InsertedNode]:
    """Inserted nodes of one iteration, in order of the call they follow.

    ``cyclic``: the iteration repeats (RLHF), so a model's last call feeds
    its first call of the next iteration (the parameter_version edge,
    SPEC.md:201) and may need a reallocation there too."""
    names = [c.name for c in calls]
    if len(set(names)) != len(names):
        raise ValueError("call names must be unique")
    by_name = {c.name: c for c in calls}
    for c in calls:
        if c.model not in models:
            raise ValueError(f"call {c.name!r}: unknown model {c.model!r}")
    out: List[InsertedNode] = []
    order = {c.name: i for i, c in enumerate(calls)}
    per_model: Dict[str, List[Call]] = {}
    for c in calls:
        per_model.setdefault(c.model, []).append(c)
    for model, seq in per_model.items():
        spec = models[model]
        pairs = list(zip(seq, seq[1:]))
        if cyclic and len(seq) > 0:
            pairs.append((seq[-1], seq[0]))
        for a, b in pairs:
            if a is b:
                # a single call per iteration: parked parameters still travel
                if a.offload:
                    out.extend(_park(spec, a, b, cluster, profile))
                continue
            if a.offload:
                out.extend(_park(spec, a, b, cluster, profile))
            if _same(a.placement, b.placement):
                continue
            plan = plan_param_realloc(spec, a.placement, b.placement, cluster, policy)
            est = costmodel.estimate_seconds(plan, profile=profile)
            out.append(InsertedNode("param_realloc", (a.name, b.name), model, plan.total_bytes, plan.est_time,
                                    est["seconds"], plan))
    for e in edges:
        if e.producer not in by_name or e.consumer not in by_name:
            raise ValueError(f"data edge {e.producer!r} -> {e.consumer!r}: unknown call")
        p, q = by_name[e.producer].placement, by_name[e.consumer].placement
        if _grid(p) == _grid(q):
            continue
        plan = plan_data_transfer(p, q, e.bytes_per_dp_shard, cluster, policy)
        est = costmodel.estimate_seconds(plan, profile=profile)
        out.append(InsertedNode("data_transfer", (e.producer, e.consumer), None, plan.total_bytes, plan.est_time,
                                est["seconds"], plan))
    out.sort(key=lambda n: (order[n.between[0]], n.kind != "offload"))
    return out


def _park(spec: ModelSpec, a: Call, b: Call, cluster: ClusterSpec,
          profile: costmodel.B200Profile) -> List[InsertedNode]:
    """Offload after call a, onload before call b (param bytes /
    host_to_device_bw). The parked shards are a's layout; a reallocation to
    b's layout, if any, follows the onload (rr_exec_launch_onload pipelines
    the two). Every GPU parks its own shard over its own host link, so the
    per-GPU shard bytes set the duration."""
    pa = plan_param_realloc(spec, a.placement, a.placement, cluster)
    nbytes = _shard_max(pa, 0)
    return [InsertedNode(kind, (a.name, b.name), a.model, nbytes, nbytes / cluster.host_to_device_bw,
                         costmodel.host_transfer_seconds(nbytes, profile))
            for kind in ("offload", "onload")]


def total_seconds(nodes: Sequence[InsertedNode]) -> Dict[str, float]:
    """Serial sum of the inserted nodes under both estimates (an upper
    bound on what they add to an iteration; the simulator overlaps them)."""
    return {"spec_seconds": sum(n.spec_seconds for n in nodes), "b200_seconds": sum(n.b200_seconds for n in nodes)}
