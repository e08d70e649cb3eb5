"""Copy-engine runs (rr_plan_ce_runs, capi_exec.cpp ce_runs): ranges moved
whole by a copy engine must be byte-identical between the source shard and
the destination shard they are copied into, and must carry (almost) only
bytes the plan moves between that pair. Checked on CPU against the oracle's
shard contents (oracle/realloc_oracle.c orc_fill)."""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest

from _helpers import placement
from oracle import oracle as O
from paper_2406_14088_b200.rlplan import BALANCED, MODELS, b200_cluster, plan_param_realloc

TINY_GQA = dataclasses.replace(MODELS["tiny"], name="tiny_gqa", hidden_size=512, num_attention_heads=16,
                               num_kv_heads=8, intermediate_size=1024)


def _hosts(n_dev: int, world: int):
    return [d * world // n_dev for d in range(n_dev)]


@pytest.mark.parametrize("sp,dp,world", [
    ((2, 1, 4, 0, 0), (1, 2, 4, 0, 0), 2),   # 13B-style pipeline-stage remap
    ((2, 1, 4, 0, 0), (1, 2, 4, 0, 0), 4),
    ((2, 1, 4, 0, 0), (1, 2, 4, 0, 0), 8),
    ((2, 2, 2, 1, 1), (1, 4, 2, 1, 1), 4),   # fused QKV / gate-up on both sides, dp replicas
    ((1, 1, 8, 0, 0), (1, 8, 1, 0, 0), 2),   # tp -> dp: no run may appear
    ((2, 1, 4, 0, 0), (1, 1, 8, 0, 0), 2),   # tp split changes: no run
])
def test_runs_are_byte_identical(sp, dp, world):
    c = b200_cluster(8)
    src = placement(8, *sp[:3], qkv=sp[3], gate_up=sp[4])
    dst = placement(8, *dp[:3], qkv=dp[3], gate_up=dp[4])
    plan = plan_param_realloc(TINY_GQA, src, dst, c, BALANCED)
    host_of = _hosts(8, world)
    seed = 5
    fills_s, fills_d = {}, {}
    total = 0
    for r in range(world):
        local = [d for d in range(8) if host_of[d] == r]
        for (s, d, so, do, nb) in plan.ce_runs(local, host_of, min_run_bytes=4096):
            assert host_of[s] == r and host_of[d] != r, "runs go from a local source to a remote destination"
            if s not in fills_s:
                fills_s[s] = O.fill(TINY_GQA, src, c, s, seed).view(np.uint8)
            if d not in fills_d:
                fills_d[d] = O.fill(TINY_GQA, dst, c, d, seed).view(np.uint8)
            a, b = fills_s[s], fills_d[d]
            assert so + nb <= a.size and do + nb <= b.size
            assert np.array_equal(a[so:so + nb], b[do:do + nb]), (s, d, so, do, nb)
            total += nb
    if sp[2] != dp[2]:
        assert total == 0, "a TP change leaves no identically laid-out range"
    else:
        # every cross-host byte of a pure stage remap goes through runs
        wire = sum(plan.work([d for d in range(8) if host_of[d] == r], 0, host_of)["wire_in"] for r in range(world))
        assert total >= 0.98 * wire, (total, wire)


@pytest.mark.parametrize("world,expect", [(2, 4 * 4), (4, 6 * 4), (8, 7 * 4)])
def test_stage_slots_7b_all_gather(world, expect):
    """Staged gather (rr_plan_stage_slots): every host receives the tp8
    source shards it does not hold, each in ceil(2.008 GB / 512 MiB) = 4
    pieces."""
    from paper_2406_14088_b200 import runtime as R
    from paper_2406_14088_b200.workloads import WORKLOADS
    w = WORKLOADS["llama7b_tp8_dp8_roundtrip"]
    plan = plan_param_realloc(w.model, *w.phases[0], w.cluster(), BALANCED)
    host_of = _hosts(8, world)
    # piece slots, then one round token per host (+1) for the aligned rounds
    assert R.stage_slots(plan, host_of, 512 << 20) == expect + world + 1
    # the gen -> train phase reads only local replicas: nothing to stage
    back = plan_param_realloc(w.model, *w.phases[1], w.cluster(), BALANCED)
    assert R.stage_slots(back, host_of, 512 << 20) == world + 1


@pytest.mark.parametrize("world", [4, 8])
def test_staged_auto_policy(world):
    """RankRealloc(staged="auto") stages only all-gather-shaped phases whose
    receivers read whole remote shards (7B tp8 -> dp8), never the partial
    TP-change reads of 34B/70B (whole shards would cross the links 2-4x),
    stage remaps (copy-engine runs), single-source broadcasts or small data
    phases."""
    from paper_2406_14088_b200 import runtime as R
    from paper_2406_14088_b200.workloads import WORKLOADS
    host_of = _hosts(8, world)
    picked = {name: [R._all_gather_shaped(p, host_of, world) for p in w.plans(BALANCED)]
              for name, w in WORKLOADS.items() if w.devices == 8}
    assert picked.pop("llama7b_tp8_dp8_roundtrip") == [True, False]
    assert not any(any(v) for v in picked.values()), picked
