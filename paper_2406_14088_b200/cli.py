"""Command line: the reference CLI's ``realloc-plan`` subcommand (SPEC.md:642,
SPEC.md:604) plus ``data-plan`` and the simulator's
``augment`` step, over the B200 planner.

    python -m paper_2406_14088_b200 realloc-plan CONFIG.json [-o PLAN.json]
    python -m paper_2406_14088_b200 data-plan CONFIG.json [-o PLAN.json]
    python -m paper_2406_14088_b200 augment PLAN.json [-o NODES.json]

``augment`` takes {"schema": 1, "cluster": ..., "models": {handle: preset or
object}, "calls": [{"name", "model", "placement": {...}, "offload"}],
"edges": [{"producer", "consumer", "bytes_per_dp_shard"}], "cyclic": true}
and prints the inserted param_realloc / data_transfer / offload / onload
nodes with the SPEC and measured-B200 durations.

CONFIG (single JSON file, schema version 1, no environment variables —
SPEC.md:657):

    {"schema": 1,
     "cluster": {"n_nodes": 1, "gpus_per_node": 8, "mem_per_device": 192265846784,
                 "intra_node_bw": 9e11, "inter_node_bw": 5e10, "host_to_device_bw": 5.5e10},
     "model": "llama7b"  |  {"name": ..., "hidden_size": ..., ...},
     "src": {"mesh": "trainer01", "dp": 1, "tp": 8, "pp": 1, "qkv_layout": "separate",
             "gate_up_layout": "separate", "kv_layout": "split" | "replicate"},
     "dst": {"mesh": "trainer01", "dp": 8, "tp": 1, "pp": 1},
     "policy": "spec" | "balanced",
     "gpus_per_host": 1,                      (plan devices per GPU, cost model)
     "data_bytes_per_dp_shard": 1048576}      (data-plan only)

Output: the plan JSON (op list with src, dst set, layer range, slice index,
bytes) extended with per-device traffic and the measured B200
time estimate (costmodel.py) beside the SPEC bytes/bandwidth estimate. Exit
code 0 iff no error; errors name the offending config path.
"""
from __future__ import annotations

import argparse
import json
import sys
from typing import Any, Dict

from . import costmodel
from .rlplan import (BALANCED, MODELS, SPEC, ClusterSpec, ModelSpec, ParallelStrategy, Placement,
                     ValidationError, mesh_from_string, plan_data_transfer, plan_param_realloc)

QKV = {"separate": 0, "concat": 1, "grouped": 2}
GATE_UP = {"separate": 0, "concat": 1}
KV = {"split": 0, "replicate": 1}


class ConfigError(ValueError):
    pass


def _get(d: Dict[str, Any], key: str, path: str, kind=None, default=None):
    if key not in d:
        if default is not None:
            return default
        raise ConfigError(f"{path}.{key}: missing")
    v = d[key]
    if kind is not None and not isinstance(v, kind):
        raise ConfigError(f"{path}.{key}: expected {getattr(kind, '__name__', kind)}")
    return v


def parse_cluster(d, path="$.cluster") -> ClusterSpec:
    if not isinstance(d, dict):
        raise ConfigError(f"{path}: expected an object")
    c = ClusterSpec(n_nodes=_get(d, "n_nodes", path, int), gpus_per_node=_get(d, "gpus_per_node", path, int),
                    mem_per_device=_get(d, "mem_per_device", path, int),
                    intra_node_bw=float(_get(d, "intra_node_bw", path, (int, float))),
                    inter_node_bw=float(_get(d, "inter_node_bw", path, (int, float))),
                    host_to_device_bw=float(_get(d, "host_to_device_bw", path, (int, float))))
    try:
        c.validate()
    except ValidationError as e:
        raise ConfigError(f"{path}: {e}") from None
    return c


def parse_model(v, path="$.model") -> ModelSpec:
    if isinstance(v, str):
        if v not in MODELS:
            raise ConfigError(f"{path}: unknown preset {v!r} (known: {', '.join(sorted(MODELS))})")
        return MODELS[v]
    if not isinstance(v, dict):
        raise ConfigError(f"{path}: expected a preset name or an object")
    fields = ModelSpec.__dataclass_fields__
    unknown = set(v) - set(fields)
    if unknown:
        raise ConfigError(f"{path}: unknown fields {sorted(unknown)}")
    m = ModelSpec(**v)
    try:
        m.validate()
    except ValidationError as e:
        raise ConfigError(f"{path}: {e}") from None
    return m


def parse_placement(d, cluster: ClusterSpec, path: str) -> Placement:
    if not isinstance(d, dict):
        raise ConfigError(f"{path}: expected an object")
    try:
        mesh = mesh_from_string(_get(d, "mesh", path, str), cluster)
    except ValidationError as e:
        raise ConfigError(f"{path}.mesh: {e}") from None
    qkv = _get(d, "qkv_layout", path, str, "separate")
    gu = _get(d, "gate_up_layout", path, str, "separate")
    if qkv not in QKV:
        raise ConfigError(f"{path}.qkv_layout: one of {sorted(QKV)}")
    if gu not in GATE_UP:
        raise ConfigError(f"{path}.gate_up_layout: one of {sorted(GATE_UP)}")
    kv = _get(d, "kv_layout", path, str, "split")
    if kv not in KV:
        raise ConfigError(f"{path}.kv_layout: one of {sorted(KV)}")
    s = ParallelStrategy(dp=_get(d, "dp", path, int), tp=_get(d, "tp", path, int), pp=_get(d, "pp", path, int),
                         n_microbatches=_get(d, "n_microbatches", path, int, 1))
    return Placement(mesh, s, QKV[qkv], GATE_UP[gu], KV[kv])


def build(config: Dict[str, Any], data: bool = False) -> Dict[str, Any]:
    if not isinstance(config, dict):
        raise ConfigError("$: expected an object")
    if _get(config, "schema", "$", int) != 1:
        raise ConfigError("$.schema: only schema 1 is supported")
    cluster = parse_cluster(_get(config, "cluster", "$"))
    src = parse_placement(_get(config, "src", "$"), cluster, "$.src")
    dst = parse_placement(_get(config, "dst", "$"), cluster, "$.dst")
    pol = _get(config, "policy", "$", str, "spec")
    if pol not in ("spec", "balanced"):
        raise ConfigError("$.policy: 'spec' or 'balanced'")
    policy = SPEC if pol == "spec" else BALANCED
    try:
        if data:
            per = _get(config, "data_bytes_per_dp_shard", "$", int)
            plan = plan_data_transfer(src, dst, per, cluster, policy)
        else:
            plan = plan_param_realloc(parse_model(_get(config, "model", "$")), src, dst, cluster, policy)
    except ValidationError as e:
        raise ConfigError(f"$: {e}") from None
    out = plan.to_json()
    k = _get(config, "gpus_per_host", "$", int, 1)
    n = cluster.device_count()
    if k < 1 or n % k:
        raise ConfigError("$.gpus_per_host: must divide the cluster's device count")
    host_of = [d // k for d in range(n)]
    out["device_traffic"] = {str(d): dict(zip(("wire_in", "wire_out", "local"), plan.device_traffic(d)))
                             for d in range(n)}
    out["b200_estimate"] = costmodel.estimate_best(plan, host_of)
    return out


def build_augment(config: Dict[str, Any]) -> Dict[str, Any]:
    """``augment``: the nodes an execution plan inserts,
    each with the SPEC estimate and the measured B200 time."""
    from .augment import Call, DataEdge, augment, total_seconds
    if not isinstance(config, dict):
        raise ConfigError("$: expected an object")
    if _get(config, "schema", "$", int) != 1:
        raise ConfigError("$.schema: only schema 1 is supported")
    cluster = parse_cluster(_get(config, "cluster", "$"))
    models_cfg = _get(config, "models", "$", dict)
    models = {k: parse_model(v, f"$.models.{k}") for k, v in models_cfg.items()}
    calls = []
    for i, c in enumerate(_get(config, "calls", "$", list)):
        path = f"$.calls[{i}]"
        if not isinstance(c, dict):
            raise ConfigError(f"{path}: expected an object")
        model = _get(c, "model", path, str)
        if model not in models:
            raise ConfigError(f"{path}.model: {model!r} is not in $.models")
        calls.append(Call(_get(c, "name", path, str), model,
                          parse_placement(_get(c, "placement", path), cluster, f"{path}.placement"),
                          bool(_get(c, "offload", path, bool, False))))
    edges = []
    for i, e in enumerate(_get(config, "edges", "$", list, [])):
        path = f"$.edges[{i}]"
        if not isinstance(e, dict):
            raise ConfigError(f"{path}: expected an object")
        edges.append(DataEdge(_get(e, "producer", path, str), _get(e, "consumer", path, str),
                              _get(e, "bytes_per_dp_shard", path, int)))
    pol = _get(config, "policy", "$", str, "balanced")
    if pol not in ("spec", "balanced"):
        raise ConfigError("$.policy: 'spec' or 'balanced'")
    try:
        nodes = augment(calls, edges, models, cluster, cyclic=bool(_get(config, "cyclic", "$", bool, True)),
                        policy=SPEC if pol == "spec" else BALANCED)
    except (ValidationError, ValueError) as e:
        raise ConfigError(f"$: {e}") from None
    return {"nodes": [{"kind": n.kind, "after": n.between[0], "before": n.between[1], "model": n.model,
                       "bytes": n.bytes, "spec_seconds": n.spec_seconds, "b200_seconds": n.b200_seconds}
                      for n in nodes],
            "totals": total_seconds(nodes)}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2406_14088_b200", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("realloc-plan", "data-plan", "augment"):
        p = sub.add_parser(name)
        p.add_argument("config")
        p.add_argument("-o", "--output")
    args = ap.parse_args(argv)
    try:
        with open(args.config) as f:
            config = json.load(f)
        out = build_augment(config) if args.cmd == "augment" else build(config, data=args.cmd == "data-plan")
    except (OSError, json.JSONDecodeError) as e:
        print(f"error: {args.config}: {e}", file=sys.stderr)
        return 2
    except ConfigError as e:
        print(f"error: {args.config}: {e}", file=sys.stderr)
        return 1
    text = json.dumps(out, indent=1, sort_keys=True)
    if args.output:
        with open(args.output, "w") as f:
            f.write(text + "\n")
    else:
        print(text)
    return 0
