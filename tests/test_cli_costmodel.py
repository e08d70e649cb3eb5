"""realloc-plan / data-plan CLI and the
measured B200 cost model (costmodel.py) against the round-1 measurements."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from paper_2406_14088_b200 import cli, costmodel
from paper_2406_14088_b200.rlplan import BALANCED, plan_param_realloc
from paper_2406_14088_b200.workloads import WORKLOADS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXAMPLE = os.path.join(ROOT, "examples", "llama7b_train_to_gen.json")


def run(*args):
    return subprocess.run([sys.executable, "-m", "paper_2406_14088_b200", *args], cwd=ROOT, capture_output=True,
                          text=True)


def test_realloc_plan_cli_emits_plan_json(tmp_path):
    out = tmp_path / "plan.json"
    r = run("realloc-plan", EXAMPLE, "-o", str(out))
    assert r.returncode == 0, r.stderr
    plan = json.load(open(out))
    assert len(plan["ops"]) == 8 and plan["total_bytes"] == 112419930112
    for op in plan["ops"]:
        assert {"src", "dst", "layer_range", "slice_index", "bytes"} <= set(op)
    assert plan["b200_estimate"]["seconds"] > plan["est_time"]


def test_identical_src_dst_gives_empty_op_list(tmp_path):
    """SPEC.md:649."""
    cfg = json.load(open(EXAMPLE))
    cfg["dst"] = cfg["src"]
    p = tmp_path / "same.json"
    p.write_text(json.dumps(cfg))
    r = run("realloc-plan", str(p))
    assert r.returncode == 0 and json.loads(r.stdout)["ops"] == []


@pytest.mark.parametrize("edit,path", [
    (lambda c: c["src"].update(mesh="trainer01:gpu[1-2]"), "$.src.mesh"),
    (lambda c: c["dst"].update(dp=4), "$: Placement: dp*tp*pp must equal the mesh size"),
    (lambda c: c.update(model="llama99b"), "$.model: unknown preset"),
    (lambda c: c.update(schema=2), "$.schema"),
    (lambda c: c["cluster"].pop("n_nodes"), "$.cluster.n_nodes: missing"),
])
def test_config_errors_name_the_path(tmp_path, edit, path):
    """exit code != 0, diagnostics name the offending path."""
    cfg = json.load(open(EXAMPLE))
    edit(cfg)
    p = tmp_path / "bad.json"
    p.write_text(json.dumps(cfg))
    r = run("realloc-plan", str(p))
    assert r.returncode == 1 and path in r.stderr, r.stderr


def test_data_plan_cli(tmp_path):
    cfg = json.load(open(EXAMPLE))
    cfg["src"] = {"mesh": "trainer01:gpu[0-1]", "dp": 2, "tp": 1, "pp": 1}
    cfg["dst"] = {"mesh": "trainer01:gpu[0-3]", "dp": 1, "tp": 4, "pp": 1}
    cfg["data_bytes_per_dp_shard"] = 1 << 20
    p = tmp_path / "data.json"
    p.write_text(json.dumps(cfg))
    out = cli.build(json.load(open(p)), data=True)
    assert out["total_bytes"] == 2 * (1 << 20) // 2 * 2 + 2 * (2 << 20)  # 2 holders x half + 2 empty x full


@pytest.mark.parametrize("gpus,measured_ms,tol", [
    (1, 22.79, 0.05),   # r01 forward phase, 1 GPU (HBM-bound)
    (2, 11.31, 0.05),   # r01 forward phase 0, 2 GPUs (NVLink-bound)
    (4, 17.03, 0.05),   # r01 forward phase 0, 4 GPUs
])
def test_cost_model_matches_round1_measurements(gpus, measured_ms, tol):
    w = WORKLOADS["llama7b_tp8_dp8_roundtrip"]
    plan = plan_param_realloc(w.model, *w.phases[0], w.cluster(), BALANCED)
    host_of = [d // (8 // gpus) for d in range(8)]
    est = costmodel.estimate_seconds(plan, host_of)
    assert est["phase0_s"] * 1e3 == pytest.approx(measured_ms, rel=tol)


def test_cost_model_staged_gather():
    """7B tp8->dp8 forward at 4 GPUs with the staged gather (bench default
    from 4 GPUs on): 16.25 ms measured (profiles/r01_staged_ab_n4.txt)."""
    w = WORKLOADS["llama7b_tp8_dp8_roundtrip"]
    plan = plan_param_realloc(w.model, *w.phases[0], w.cluster(), BALANCED)
    host_of = [d // 2 for d in range(8)]
    est = costmodel.estimate_seconds(plan, host_of, staged=True)
    assert est["phase0_s"] * 1e3 == pytest.approx(16.25, rel=0.05)


@pytest.mark.parametrize("gpus,measured_ms,ce", [
    (2, 18.54, True),    # 13B stage remap with copy-engine runs (profiles/r01_configs_n2.jsonl)
    (4, 9.32, True),     # (profiles/r01_configs_n4.jsonl)
    (2, 19.65, False),   # the same with SM peer stores only (profiles/r01_ce_runs_ab_n2_n4.jsonl)
    (4, 9.84, False),
])
def test_cost_model_stage_remap(gpus, measured_ms, ce):
    w = WORKLOADS["llama13b_pp2tp4_to_dp2tp4"]
    plan = plan_param_realloc(w.model, *w.phases[0], w.cluster(), BALANCED)
    host_of = [d // (8 // gpus) for d in range(8)]
    est = costmodel.estimate_seconds(plan, host_of, copy_engine=ce)
    assert est["phase0_s"] * 1e3 == pytest.approx(measured_ms, rel=0.05)


@pytest.mark.parametrize("gpus,measured_ms", [
    (1, 294.4),   # r01 bench e2e, 1 GPU (profiles/r01_bench_default_n1.json): 16.06 GB onloaded per step
    (2, 152.4),   # round-1 bench e2e at 2 GPUs, 8.03 GB onloaded per GPU
])
def test_cost_model_onload_matches_e2e(gpus, measured_ms):
    """With the sources onloaded from host memory the round trip is bound by
    each GPU's host link (SPEC.md:423 prices onload at bytes /
    host_to_device_bw); the measured rate reproduces the e2e step."""
    w = WORKLOADS["llama7b_tp8_dp8_roundtrip"]
    host_of = [d // (8 // gpus) for d in range(8)]
    fwd = costmodel.estimate_seconds(plan_param_realloc(w.model, *w.phases[0], w.cluster(), BALANCED), host_of,
                                     onload=True)
    back = costmodel.estimate_seconds(plan_param_realloc(w.model, *w.phases[1], w.cluster(), BALANCED), host_of)
    assert fwd["onload_s"] > fwd["seconds"] - fwd["onload_s"]  # host-link bound
    assert (fwd["seconds"] + back["seconds"]) * 1e3 == pytest.approx(measured_ms, rel=0.08)


def test_augment_cli_on_the_ppo_example(tmp_path):
    """`augment` over examples/ppo_7b_augment.json: one
    node per layout change, data edge and offload flag, each priced by the
    SPEC and by the measured B200 model."""
    import os
    ex = os.path.join(os.path.dirname(__file__), "..", "examples", "ppo_7b_augment.json")
    out = tmp_path / "nodes.json"
    assert cli.main(["augment", ex, "-o", str(out)]) == 0
    d = json.load(open(out))
    kinds = [n["kind"] for n in d["nodes"]]
    assert kinds.count("param_realloc") == 4 and kinds.count("data_transfer") == 6
    assert kinds.count("offload") == kinds.count("onload") == 2
    gen_to_train = next(n for n in d["nodes"] if n["kind"] == "param_realloc" and n["after"] == "ActorGen")
    # dp8 -> tp8 keeps every byte on its device: SPEC prices it at 0 s, the
    # B200 model at the local relayout's HBM time
    assert gen_to_train["bytes"] == 0 and gen_to_train["spec_seconds"] == 0 and gen_to_train["b200_seconds"] > 0
    bad = json.load(open(ex))
    bad["calls"][0]["model"] = "nobody"
    p = tmp_path / "bad.json"
    p.write_text(json.dumps(bad))
    assert cli.main(["augment", str(p)]) == 1


def test_bench_config_workload_matches_the_preset():
    """bench.py --config: a realloc-plan config with "back": true is the
    same two-phase workload as the named 7B round trip."""
    import os
    from paper_2406_14088_b200.workloads import from_config
    ex = os.path.join(os.path.dirname(__file__), "..", "examples", "llama7b_train_gen_roundtrip.json")
    w = from_config(json.load(open(ex)))
    ref = WORKLOADS["llama7b_tp8_dp8_roundtrip"]
    assert len(w.phases) == 2 and w.devices == ref.devices and w.model == ref.model
    for a, b in zip(w.plans(BALANCED), ref.plans(BALANCED)):
        assert a.total_bytes == b.total_bytes and a.num_rects() == b.num_rects()
        assert [op.src for op in a.ops] == [op.src for op in b.ops]


def test_realloc_plan_cli_replicated_kv_heads(tmp_path):
    """kv_layout "replicate" in a realloc-plan config (DESIGN.md §3 G6): an
    MQA model moved from one device to tp8 with replicated heads carries K/V
    as their own payloads, and the plan JSON says so."""
    cfg = json.load(open(os.path.join(os.path.dirname(__file__), "..", "examples", "llama7b_train_to_gen.json")))
    cfg["model"] = {"name": "mqa", "hidden_size": 512, "intermediate_size": 1024, "num_layers": 2,
                    "num_attention_heads": 8, "num_kv_heads": 1, "vocab_size": 1024, "max_position_embeddings": 256}
    cfg["src"] = {"mesh": "trainer01:gpu[0-0]", "dp": 1, "tp": 1, "pp": 1}
    cfg["dst"] = {"mesh": "trainer01", "dp": 1, "tp": 8, "pp": 1, "kv_layout": "replicate"}
    p = tmp_path / "mqa.json"
    p.write_text(json.dumps(cfg))
    out = cli.build(json.load(open(p)))
    assert out["dst"]["kv_layout"] == 1
    parts = {op.get("part") for op in out["ops"]}
    assert "kv" in parts and "no_kv" in parts
    kv_ops = [op for op in out["ops"] if op.get("part") == "kv"]
    assert len(kv_ops) == 1 and sorted(kv_ops[0]["dst"]) == list(range(1, 8))  # the one head, to every replica
    cfg["dst"]["kv_layout"] = "sideways"
    p.write_text(json.dumps(cfg))
    with pytest.raises(cli.ConfigError, match="kv_layout"):
        cli.build(json.load(open(p)))


@pytest.mark.parametrize("name,world,measured_ms,scheme", [
    ("llama70b_pp2tp4_to_tp8", 4, 46.50, "ce_transport"),   # profiles/r02_configs_n4.jsonl
    ("llama70b_pp2tp4_to_tp8", 2, 47.31, "ce_transport"),   # profiles/r02_configs_n2.jsonl
    ("llama34b_critic_pp4tp2_to_tp8", 4, 19.20, "ce_transport"),
    ("llama7b_tp8_dp8_roundtrip", 4, 16.07, "staged"),
])
def test_estimate_best_matches_round2_measurements(name, world, measured_ms, scheme):
    """The cost-model twin of the bind-time probe picks the scheme the probe
    picked on the B200s and lands within 5% of its measured phase time."""
    from paper_2406_14088_b200.workloads import WORKLOADS
    plan = WORKLOADS[name].plans(BALANCED)[0]
    est = costmodel.estimate_best(plan, [d * world // 8 for d in range(8)])
    assert est["scheme"] == scheme
    assert est["seconds"] * 1e3 == pytest.approx(measured_ms, rel=0.05)
