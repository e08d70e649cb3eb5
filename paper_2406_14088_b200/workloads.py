"""Named reallocation workloads: the BASELINE.json configs as placements.

Each workload is a list of phases (src placement -> dst placement) over the
same plan devices; a bench "step" runs every phase once. Placements are
written (pp, dp, tp) as in BASELINE.json.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

from .rlplan import (BALANCED, GATE_UP_CONCAT, GATE_UP_SEPARATE, MODELS, QKV_CONCAT, QKV_GROUPED,
                     QKV_SEPARATE, ClusterSpec, DeviceMesh, ModelSpec, ParallelStrategy, Placement,
                     ReallocPlan, b200_cluster, plan_data_transfer, plan_param_realloc)


def layout(devices: int, pp: int, dp: int, tp: int, qkv: int = QKV_SEPARATE,
           gate_up: int = GATE_UP_SEPARATE) -> Placement:
    return Placement(DeviceMesh(0, 1, 0, devices), ParallelStrategy(dp=dp, tp=tp, pp=pp), qkv, gate_up)


@dataclass(frozen=True)
class Workload:
    name: str
    description: str
    model: ModelSpec
    devices: int                      # plan devices (hosted on 1..devices GPUs)
    phases: Tuple[Tuple[Placement, Placement], ...]
    # > 0: inter-call data transfer (plan_data_transfer) of
    # this many bytes per producer DP shard instead of a parameter plan
    data_bytes: int = 0
    cluster_spec: Optional[ClusterSpec] = None  # default: one B200 node with `devices` GPUs

    def cluster(self) -> ClusterSpec:
        return self.cluster_spec or b200_cluster(self.devices)

    def plans(self, policy: int = BALANCED) -> List[ReallocPlan]:
        c = self.cluster()
        if self.data_bytes:
            return [plan_data_transfer(s, d, self.data_bytes, c, policy) for s, d in self.phases]
        return [plan_param_realloc(self.model, s, d, c, policy) for s, d in self.phases]


def _pp(p: Placement) -> str:
    s = p.strategy
    return f"(pp{s.pp},dp{s.dp},tp{s.tp})"


def _make(name: str, model: str, devices: int, src: Placement, dst: Placement, back: bool,
          desc: str) -> Workload:
    phases = ((src, dst), (dst, src)) if back else ((src, dst),)
    return Workload(name, desc, MODELS[model], devices, phases)


WORKLOADS: Dict[str, Workload] = {}


def _register(w: Workload) -> None:
    WORKLOADS[w.name] = w


# BASELINE.json configs[0]: the CPU oracle case.
_register(_make("tiny_tp2_to_dp2", "tiny", 2, layout(2, 1, 1, 2), layout(2, 1, 2, 1), False,
                "tiny LLaMA (4L, h256) (pp1,dp1,tp2)->(pp1,dp2,tp1) on 2 devices"))
# BASELINE.json configs[1]: actor train layout -> generation layout and back.
_register(_make("llama7b_tp8_dp8_roundtrip", "llama7b", 8, layout(8, 1, 1, 8), layout(8, 1, 8, 1), True,
                "LLaMA-7B bf16 train (pp1,dp1,tp8) -> gen (pp1,dp8,tp1) and back, 8 plan devices"))
# BASELINE.json configs[2]: pipeline-stage remap.
_register(_make("llama13b_pp2tp4_to_dp2tp4", "llama13b", 8, layout(8, 2, 1, 4), layout(8, 1, 2, 4), False,
                "LLaMA-13B bf16 (pp2,dp1,tp4)->(pp1,dp2,tp4)"))
# BASELINE.json configs[3]: critic with Megatron-grouped QKV / fused gate-up -> concat layouts.
_register(_make("llama34b_critic_pp4tp2_to_tp8", "llama34b_critic", 8,
                layout(8, 4, 1, 2, QKV_GROUPED, GATE_UP_CONCAT), layout(8, 1, 1, 8, QKV_CONCAT, GATE_UP_CONCAT),
                False, "LLaMA-34B critic bf16 (pp4,dp1,tp2)->(pp1,dp1,tp8), fused QKV/gate-up reinterleave"))
# BASELINE.json configs[4]: full-box 70B.
_register(_make("llama70b_pp2tp4_to_tp8", "llama70b", 8, layout(8, 2, 1, 4), layout(8, 1, 1, 8), False,
                "LLaMA-70B bf16 (pp2,dp1,tp4)->(pp1,dp1,tp8)"))


# Parameter sync of a whole replica to a DP group (disjoint =
# parameter sync): every op is a contiguous one-to-many broadcast.
_register(Workload("llama7b_replicate_to_dp8", "LLaMA-7B bf16 (pp1,dp1,tp1) on device 0 -> (pp1,dp8,tp1)",
                   MODELS["llama7b"], 8,
                   ((Placement(DeviceMesh(0, 1, 0, 1), ParallelStrategy()), layout(8, 1, 8, 1)),)))


# Inter-call data transfer (DP-partitioned outputs of one
# function call redistributed to the next call's layout). 32 MiB per
# generation DP shard is a 256 MiB batch of per-token RLHF data.
_register(Workload("data_gen_dp8_to_train_tp8",
                   "RLHF batch, 32 MiB per DP shard: actor generation (pp1,dp8,tp1) -> training (pp1,dp1,tp8)",
                   MODELS["llama7b"], 8, ((layout(8, 1, 8, 1), layout(8, 1, 1, 8)),), data_bytes=32 << 20))
_register(Workload("data_gen_dp8_to_pp2dp2tp2",
                   "RLHF batch, 32 MiB per DP shard: generation (pp1,dp8,tp1) -> critic (pp2,dp2,tp2)",
                   MODELS["llama7b"], 8, ((layout(8, 1, 8, 1), layout(8, 2, 2, 2)),), data_bytes=32 << 20))


def truncated(w: Workload, layers: int) -> Workload:
    """Same shapes and layouts with fewer decoder layers (bounded samples);
    a data workload has no layers and is returned unchanged."""
    if w.data_bytes:
        return w
    m = dataclasses.replace(w.model, num_layers=layers)
    return Workload(f"{w.name}[{layers}L]", w.description + f", truncated to {layers} layers", m, w.devices,
                    w.phases)


def from_config(config: dict, name: str = "config") -> Workload:
    """A workload from a ``realloc-plan`` / ``data-plan`` config (cli.py
    format) so any placement pair can be benchmarked: ``"back": true`` adds
    the return phase, ``data_bytes_per_dp_shard`` makes it a data transfer.
    The plan devices are the cluster's devices."""
    from .cli import ConfigError, _get, parse_cluster, parse_model, parse_placement
    if _get(config, "schema", "$", int) != 1:
        raise ConfigError("$.schema: only schema 1 is supported")
    cluster = parse_cluster(_get(config, "cluster", "$"))
    if cluster.n_nodes != 1:
        raise ConfigError("$.cluster.n_nodes: execution is single-node (CUDA IPC between the node's GPUs)")
    src = parse_placement(_get(config, "src", "$"), cluster, "$.src")
    dst = parse_placement(_get(config, "dst", "$"), cluster, "$.dst")
    back = bool(_get(config, "back", "$", bool, False))
    data = int(_get(config, "data_bytes_per_dp_shard", "$", int, 0))
    model = MODELS["tiny"] if data else parse_model(_get(config, "model", "$"))
    phases = ((src, dst), (dst, src)) if back else ((src, dst),)
    desc = f"{model.name if not data else 'data'} {_pp(src)} -> {_pp(dst)}" + (" and back" if back else "")
    return Workload(name, desc, model, cluster.device_count(), phases, data_bytes=data, cluster_spec=cluster)
