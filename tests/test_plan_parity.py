"""Planner parity: product plan_param_realloc (C++ behind the C ABI) vs the
oracle's independent C restatement of SPEC.md:569-577, the SPEC examples,
the SPEC invariants and the replay criterion (SPEC.md:577,
acceptance criterion 6 at SPEC.md:679)."""
from __future__ import annotations

import dataclasses
import random
import time

import pytest

from _helpers import BASELINE_CONFIGS, config_placements, op_tuple, placement, random_placement
from oracle import oracle as O
from paper_2406_14088_b200 import rlplan as P
from paper_2406_14088_b200.rlplan import BALANCED, SPEC

TINY_GQA = dataclasses.replace(P.MODELS["tiny"], name="tiny_gqa", hidden_size=512, num_attention_heads=16,
                               num_kv_heads=8, intermediate_size=1024)


def both(model, src, dst, c, policy):
    p = P.plan_param_realloc(model, src, dst, c, policy)
    o = O.plan(model, src, dst, c, policy)
    assert o is not None
    ops, loc, tb, et = o
    assert [op_tuple(x) for x in p.ops] == ops
    assert [op_tuple(x) for x in p.local_ops] == loc
    assert p.total_bytes == tb
    assert p.est_time == pytest.approx(et, rel=1e-12)
    return p, ops, loc


def model_bytes(m):
    return P.natural_param_count(m) * m.param_bytes


def check_invariants(m, src, dst, c, p):
    # SPEC.md:589-592
    n_dst = len(dst.mesh.devices(c))
    assert 0 <= p.total_bytes <= n_dst * model_bytes(m)
    assert (p.total_bytes == 0) == (len(p.ops) == 0)
    assert (p.est_time == 0) == (p.total_bytes == 0)
    for op in p.ops:
        assert op.src not in op.dst
        assert op.bytes > 0
    # every delivered byte is accounted for exactly once per destination
    delivered = sum(op.bytes * len(op.dst) for op in p.ops) + sum(op.bytes * len(op.dst) for op in p.local_ops)
    assert delivered == sum(p.shard_bytes(1, d) - _padding(p, 1, d) for d in dst.mesh.devices(c))


def _padding(plan, side, d):
    blocks = plan.layout(side, d)
    used = sum((b[2] - b[1]) * (b[4] - b[3]) * 2 for b in blocks)
    return plan.shard_bytes(side, d) - used


def test_spec_identical_placements_empty_plan():
    """src == dst -> no ops, 0 bytes, 0 s."""
    for key in BASELINE_CONFIGS:
        m, src, _dst, c = config_placements(key)
        for policy in (SPEC, BALANCED):
            p, ops, _loc = both(m, src, src, c, policy)
            assert p.ops == [] and p.total_bytes == 0 and p.est_time == 0.0
            assert p.to_json()["ops"] == []


def test_spec_one_device_to_tp2():
    """one device holding everything -> tp2 mesh containing it:
    the own half stays local, the other half goes out in one broadcast (the
    replicated norms travel as their own payload, G5)."""
    m = P.MODELS["spec_tiny"]
    c = P.b200_cluster(2)
    src = placement(1, 1, 1, 1)
    dst = placement(2, 1, 1, 2)
    p, ops, loc = both(m, src, dst, c, SPEC)
    split = [op for op in p.ops if not op.payload.replicated]
    assert len(split) == 1 and split[0].src == 0 and split[0].dst == (1,)
    assert (split[0].payload.tp_rank, split[0].payload.tp_degree) == (1, 2)
    total = model_bytes(m)
    rep_bytes = sum(op.bytes for op in p.ops if op.payload.replicated)
    # 472 B model: 224 B split half + 24 B replicated norms
    assert total == 472 and split[0].bytes == 224 and rep_bytes == 24
    assert all(op.src == 0 and op.dst == (0,) for op in p.local_ops)
    assert O.replay(m, src, dst, c, ops, loc) is None


# SURVEY.md §8(d) / BASELINE.md derived bottleneck bytes (lowest-index sources).
DERIVED_BOTTLENECK = {
    "tiny_tp2_to_dp2": 3424256,
    "7b_tp8_to_dp8": 14052491264,
    "13b_pp2tp4_to_dp2tp4": 3501957120,
    "34b_pp4tp2_to_tp8_fused": 9355395072,
    "70b_pp2tp4_to_tp8": 17643405312,
}


@pytest.mark.parametrize("key", sorted(BASELINE_CONFIGS))
@pytest.mark.parametrize("policy", [SPEC, BALANCED])
def test_baseline_configs_plan_parity(key, policy):
    m, src, dst, c = config_placements(key)
    t = time.perf_counter()
    p, ops, loc = both(m, src, dst, c, policy)
    assert time.perf_counter() - t < 5
    assert O.replay(m, src, dst, c, ops, loc) is None
    check_invariants(m, src, dst, c, p)
    if key in DERIVED_BOTTLENECK and policy == SPEC:
        worst = max(max(p.device_traffic(d)[:2]) for d in range(c.device_count()))
        assert worst == DERIVED_BOTTLENECK[key]
    if key == "7b_dp8_to_tp8":
        assert p.ops == [] and p.total_bytes == 0  # every slice already on its own replica


def test_balanced_policy_spreads_egress():
    """dp4 on GPUs 0-3 -> tp4 on 4-7. SPEC tie-break funnels all
    egress through GPU 0; the balanced policy spreads it evenly."""
    m = P.MODELS["llama7b"]
    c = P.b200_cluster(8)
    src = placement(4, 1, 4, 1, offset=0)
    dst = placement(4, 1, 1, 4, offset=4)
    spec = P.plan_param_realloc(m, src, dst, c, SPEC)
    bal = P.plan_param_realloc(m, src, dst, c, BALANCED)
    out_spec = [spec.device_traffic(d)[1] for d in range(4)]
    out_bal = [bal.device_traffic(d)[1] for d in range(4)]
    assert out_spec[0] == sum(out_spec)
    assert max(out_bal) - min(out_bal) <= max(op.bytes for op in bal.ops)
    assert spec.total_bytes == bal.total_bytes
    assert bal.est_time < spec.est_time / 3


def test_random_placement_pairs_replay_exact():
    """SPEC.md:679 acceptance criterion 6: >= 500 random (src, dst) pairs on
    <= 8 devices replay exactly; identical placements yield 0 bytes; < 30 s."""
    rng = random.Random(2406)
    c = P.b200_cluster(8)
    models = [TINY_GQA, dataclasses.replace(TINY_GQA, num_layers=5, has_output_head=False),
              dataclasses.replace(P.MODELS["tiny"], num_layers=3)]
    t0 = time.perf_counter()
    n = 0
    while n < 520:
        m = rng.choice(models)
        src = random_placement(rng, m)
        dst = random_placement(rng, m)
        policy = rng.choice([SPEC, BALANCED])
        p, ops, loc = both(m, src, dst, c, policy)
        assert O.replay(m, src, dst, c, ops, loc) is None, (src, dst, policy)
        check_invariants(m, src, dst, c, p)
        same = P.plan_param_realloc(m, src, src, c, policy)
        assert same.total_bytes == 0 and same.ops == []
        n += 1
    assert time.perf_counter() - t0 < 30


def test_invalid_placements_raise_validation_error():
    m = P.MODELS["llama7b"]
    c = P.b200_cluster(8)
    ok = placement(8, 1, 1, 8)
    bad = [placement(8, 1, 2, 8),                      # dp*tp*pp != mesh size
           placement(8, 1, 8, 1, offset=1),             # mesh exceeds node
           P.Placement(P.DeviceMesh(0, 1, 0, 8), P.ParallelStrategy(dp=1, tp=8, pp=1), 7, 0)]
    for b in bad:
        with pytest.raises(P.ValidationError):
            P.plan_param_realloc(m, ok, b, c)
        assert O.plan(m, ok, b, c) is None
    with pytest.raises(P.ValidationError, match="pp must not exceed num_layers"):
        P.validate_placement(P.MODELS["tiny"], placement(8, 8, 1, 1), c)
    with pytest.raises(P.ValidationError, match="tp must divide num_attention_heads"):
        P.validate_placement(P.MODELS["tiny"], placement(8, 1, 1, 8), c)
    with pytest.raises(P.ValidationError, match="stage_layer_map: pp must not exceed num_layers"):
        P.stage_layer_map(3, 4)


def test_plan_json_export():
    """op list with src, dst set, layer range, slice index, bytes."""
    m, src, dst, c = config_placements("13b_pp2tp4_to_dp2tp4")
    p = P.plan_param_realloc(m, src, dst, c, SPEC)
    j = p.to_json()
    assert j["total_bytes"] == p.total_bytes and j["src"]["mesh"] == "trainer01"
    assert len(j["ops"]) == len(p.ops)
    for e, op in zip(j["ops"], p.ops):
        assert (e["src"], tuple(e["dst"]), tuple(e["layer_range"]), e["slice_index"], e["slice_count"],
                e["bytes"]) == (op.src, op.dst, (op.payload.layer_start, op.payload.layer_end),
                                op.payload.tp_rank, op.payload.tp_degree, op.bytes)


KV_MODELS = [dataclasses.replace(P.MODELS["tiny"], name="tiny_mqa", hidden_size=512, num_attention_heads=8,
                                 num_kv_heads=1, intermediate_size=1024, num_layers=3),
             dataclasses.replace(P.MODELS["tiny"], name="tiny_kv2", hidden_size=512, num_attention_heads=8,
                                 num_kv_heads=2, intermediate_size=1024, num_layers=2)]


def test_replicated_kv_heads_plans_match_oracle_and_replay():
    """DESIGN.md §3 G6 ReplicateHeads: with tp > kv heads every rank holds a
    whole KV head, so K/V travel as their own payloads (part 2) at lcm of
    the two sides' K/V slicings while everything else keeps the SPEC lcm(tp)
    slicing (part 1). 300 random pairs on MQA / 2-KV-head models: the product
    equals the oracle restatement, replay is exact, and some K/V payloads
    fan out to several replicas of a head."""
    rng = random.Random(679)
    c = P.b200_cluster(8)
    kv_ops = multi = 0
    for _ in range(300):
        m = rng.choice(KV_MODELS)
        src, dst = random_placement(rng, m), random_placement(rng, m)
        policy = rng.choice([SPEC, BALANCED])
        p, ops, loc = both(m, src, dst, c, policy)
        assert O.replay(m, src, dst, c, ops, loc) is None, (src, dst, policy)
        check_invariants(m, src, dst, c, p)
        kv = [op for op in p.ops + p.local_ops if op.payload.part == P.PART_KV]
        kv_ops += len(kv)
        multi += sum(len(op.dst) > 1 for op in kv)
    assert kv_ops > 100 and multi > 10


def test_kv_layout_validation_and_bytes():
    m = KV_MODELS[1]  # 2 KV heads
    c = P.b200_cluster(8)
    rep = dataclasses.replace(placement(8, 1, 1, 8), kv_layout=P.KV_REPLICATE_HEADS)
    split = placement(8, 1, 1, 8)
    one = placement(1, 1, 1, 1)
    # every tp8 rank of the replicated layout holds a whole head: 4x the K/V bytes of the split layout
    kv_rows = m.num_kv_heads * m.head_dim()
    p_rep = P.plan_param_realloc(m, one, rep, c)
    p_split = P.plan_param_realloc(m, one, split, c)
    extra = sum(op.bytes * len(op.dst) for op in p_rep.ops) - sum(op.bytes * len(op.dst) for op in p_split.ops)
    assert extra == m.num_layers * 2 * (kv_rows // 2 - kv_rows // 8) * m.hidden_size * 2 * 7
    # split <-> replicated on the same mesh only moves K/V rows
    p = P.plan_param_realloc(m, split, rep, c)
    assert {op.payload.part for op in p.ops} == {P.PART_KV}
    bad = dataclasses.replace(placement(8, 1, 1, 8), kv_layout=P.KV_REPLICATE_HEADS)
    with pytest.raises(P.ValidationError, match="multiple of num_kv_heads"):
        P.validate_placement(dataclasses.replace(m, num_kv_heads=3, num_attention_heads=24, hidden_size=768), bad, c)
