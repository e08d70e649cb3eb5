"""Named reallocation workloads: the BASELINE.json configs as placements.

Each workload is a list of phases (src placement -> dst placement) over the
same plan devices; a bench "step" runs every phase once. Placements are
written (pp, dp, tp) as in BASELINE.json.
"""
from __future__ import annotations

import dataclasses
import json
import os
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

from .rlplan import (BALANCED, GATE_UP_SEPARATE, MODELS, QKV_SEPARATE, ClusterSpec, DeviceMesh, ModelSpec,
                     ParallelStrategy, Placement, ReallocPlan, b200_cluster, plan_data_transfer,
                     plan_param_realloc)


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


# The named workloads live in workloads.json as plain data (BASELINE.json
# configs[0..4] and companions), so that bench.py's reference arm can build
# the very same workloads without importing this package.
TABLE_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "workloads.json")


def _placement(d: dict) -> Placement:
    no, nc, go, gc = d["mesh"]
    return Placement(DeviceMesh(no, nc, go, gc), ParallelStrategy(dp=d["dp"], tp=d["tp"], pp=d["pp"]),
                     d.get("qkv_layout", QKV_SEPARATE), d.get("gate_up_layout", GATE_UP_SEPARATE),
                     d.get("kv_layout", 0))


def _load_table() -> Dict[str, Workload]:
    with open(TABLE_PATH) as f:
        table = json.load(f)
    for name, dims in table["models"].items():  # the table restates rlplan.MODELS; keep them one
        m = MODELS[name]
        if any(getattr(m, k) != v for k, v in dims.items()):
            raise ValueError(f"workloads.json model {name!r} differs from rlplan.MODELS")
    out: Dict[str, Workload] = {}
    for e in table["workloads"]:
        src, dst = _placement(e["src"]), _placement(e["dst"])
        phases = ((src, dst), (dst, src)) if e["back"] else ((src, dst),)
        out[e["name"]] = Workload(e["name"], e["description"], MODELS[e["model"]], e["devices"], phases,
                                  data_bytes=e.get("data_bytes", 0))
    return out


WORKLOADS: Dict[str, Workload] = _load_table()


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
