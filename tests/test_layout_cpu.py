"""CPU-side parity of the layout contract and the product's lowering.

The product lowers a plan to copy rectangles by intersecting layout blocks
(paper_2406_14088_b200/csrc/planner.cpp); the oracle addresses every element
through per-tensor address functions (oracle/realloc_oracle.c). Applying the
product's rectangles with numpy to oracle-filled source shards must give
exactly the oracle's expected destination shards, and the oracle's own CPU
reallocation must agree too. The GPU tests run the same rectangles through
the sm_100a kernels."""
from __future__ import annotations

import dataclasses
import json
import os

import numpy as np
import pytest

from _helpers import BASELINE_CONFIGS, config_placements, emulate_lowered, placement
from oracle import oracle as O
from paper_2406_14088_b200 import rlplan as P
from paper_2406_14088_b200._lib import lib
from paper_2406_14088_b200.rlplan import BALANCED, SPEC

HERE = os.path.dirname(os.path.abspath(__file__))
TINY_GQA = dataclasses.replace(P.MODELS["tiny"], name="tiny_gqa", hidden_size=512, num_attention_heads=16,
                               num_kv_heads=8, intermediate_size=1024)

CASES = [
    ((1, 1, 2, 0, 0), (1, 2, 1, 0, 0), 2),
    ((1, 1, 8, 0, 0), (1, 8, 1, 0, 0), 8),
    ((1, 8, 1, 0, 0), (1, 1, 8, 0, 0), 8),
    ((4, 1, 2, 2, 1), (1, 1, 8, 1, 1), 8),
    ((2, 1, 4, 2, 1), (1, 2, 4, 0, 0), 8),
    ((1, 2, 4, 1, 0), (2, 1, 4, 2, 1), 8),
    ((1, 8, 1, 2, 1), (4, 1, 2, 0, 0), 8),
    ((2, 1, 4, 0, 0), (1, 1, 8, 0, 0), 8),
    ((2, 2, 2, 1, 1), (2, 1, 4, 2, 0), 8),
]


def weight_kat_cases():
    return json.load(open(os.path.join(HERE, "golden", "weights_kat.json")))["cases"]


def test_weight_value_known_answers():
    """The product's value function (used by the GPU fill/verify kernels, shared
    __host__ __device__ code) equals the oracle's, against frozen KATs."""
    for seed, tensor, idx, want in weight_kat_cases():
        assert O.value(seed, tensor, idx) == want
        assert lib.rr_weight_value(seed, tensor, idx) == want


def test_weight_values_are_finite_normal_bf16():
    vals = np.array([O.value(3, t, i) for t in range(4) for i in range(2000)], dtype=np.uint16)
    exp = (vals >> 7) & 0xFF
    assert exp.min() >= 117 and exp.max() <= 124
    assert len(np.unique(vals)) > 1500


@pytest.mark.parametrize("sp,dp,gpus", CASES)
@pytest.mark.parametrize("policy", [SPEC, BALANCED])
def test_lowered_rectangles_reproduce_oracle(sp, dp, gpus, policy):
    m = TINY_GQA if gpus == 8 else P.MODELS["tiny"]
    c = P.b200_cluster(gpus)
    src = placement(gpus, *sp[:3], qkv=sp[3], gate_up=sp[4])
    dst = placement(gpus, *dp[:3], qkv=dp[3], gate_up=dp[4])
    plan = P.plan_param_realloc(m, src, dst, c, policy)
    seed = 9
    sbufs = {d: O.fill(m, src, c, d, seed) for d in plan.devices(0)}
    dbufs = {d: np.zeros(plan.shard_bytes(1, d) // 2, np.uint16) for d in plan.devices(1)}
    emulate_lowered(plan, sbufs, dbufs)
    for d in plan.devices(1):
        assert np.array_equal(dbufs[d], O.fill(m, dst, c, d, seed)), f"device {d}"
    # the oracle's CPU reallocation of its own plan agrees
    ops, loc, _tb, _et = O.plan(m, src, dst, c, policy)
    n = c.device_count()
    s_list = [sbufs.get(d) for d in range(n)]
    d_list = [np.zeros(O.shard_bytes(m, dst, c, d) // 2, np.uint16) if d in dbufs else None for d in range(n)]
    O.execute(m, src, dst, c, ops + loc, s_list, d_list, 3)
    for d in plan.devices(1):
        assert np.array_equal(d_list[d], dbufs[d])


@pytest.mark.parametrize("key", sorted(BASELINE_CONFIGS))
def test_layout_tables_agree_with_oracle(key):
    """Shard sizes agree, blocks tile each shard without overlap, and the
    product's block table addresses the same bytes the oracle fills."""
    m, src, dst, c = config_placements(key)
    plan = P.plan_param_realloc(m, src, dst, c, BALANCED)
    inv_cols = {}
    for side, pl in ((0, src), (1, dst)):
        for d in plan.devices(side):
            assert plan.shard_bytes(side, d) == O.shard_bytes(m, pl, c, d)
            blocks = plan.layout(side, d)
            spans = sorted((b[5], b[5] + (b[2] - b[1]) * (b[4] - b[3]) * 2) for b in blocks)
            for (a0, a1), (b0, _b1) in zip(spans, spans[1:]):
                assert a1 <= b0
            assert spans[-1][1] <= plan.shard_bytes(side, d)
    # sampled element check on the first destination device of small configs
    if P.natural_param_count(m) < 10**8:
        d = plan.devices(1)[0]
        buf = O.fill(m, dst, c, d, 4)
        for (t, r0, r1, c0, c1, off) in plan.layout(1, d):
            cols = None
            for (rr, cc) in ((r0, c0), (r1 - 1, c1 - 1)):
                full_cols = _tensor_cols(m, t)
                idx = rr * full_cols + cc
                pos = (off + ((rr - r0) * (c1 - c0) + (cc - c0)) * 2) // 2
                assert buf[pos] == O.value(4, t, idx)
            del cols


def _tensor_cols(m, t):
    L = m.num_layers
    h = m.hidden_size
    if t == 0 or t >= 1 + 9 * L:
        return h
    kind = (t - 1) % 9
    if kind == 4:
        return m.num_attention_heads * m.head_dim()
    if kind == 8:
        return m.intermediate_size
    return h


def test_lowering_is_compact():
    """Contiguous runs are merged: the 7B tp8->dp8 plan lowers to a few
    thousand rectangles, not one per row."""
    m, src, dst, c = config_placements("7b_tp8_to_dp8")
    plan = P.plan_param_realloc(m, src, dst, c, BALANCED)
    assert plan.num_rects() < 4000
    w = plan.work(list(range(8)), 0)
    read, written = w["read"], w["written"]
    # one read of each source slice, eight stores (seven replicas + own); the
    # replicated norms are taken by every replica from itself
    assert read < written / 7.9
    assert written == sum(plan.shard_bytes(1, d) for d in range(8)) - sum(
        plan.shard_bytes(1, d) - sum((b[2] - b[1]) * (b[4] - b[3]) * 2 for b in plan.layout(1, d)) for d in range(8))


def test_random_pairs_lowering_reproduces_oracle():
    """Fuzz on CPU: the product's copy rectangles for 100 random placement
    pairs (sub-meshes, every layout, both policies) applied with numpy give
    the oracle's destination shards exactly (the GPU fuzz runs the same
    generator through the kernels)."""
    import random

    from _helpers import random_placement
    rng = random.Random(5150)
    c = P.b200_cluster(8)
    models = [TINY_GQA, dataclasses.replace(TINY_GQA, num_layers=5, has_output_head=False),
              dataclasses.replace(P.MODELS["tiny"], num_layers=3),
              # 1 and 2 KV heads: replicated-head layouts (G6) at tp > kv
              dataclasses.replace(TINY_GQA, name="tiny_mqa", num_attention_heads=8, num_kv_heads=1, num_layers=3),
              dataclasses.replace(TINY_GQA, name="tiny_kv2", num_attention_heads=8, num_kv_heads=2, num_layers=2)]
    for i in range(100):
        m = rng.choice(models)
        src, dst = random_placement(rng, m), random_placement(rng, m)
        plan = P.plan_param_realloc(m, src, dst, c, rng.choice([SPEC, BALANCED]))
        sbufs = {d: O.fill(m, src, c, d, i) for d in plan.devices(0)}
        dbufs = {d: np.zeros(plan.shard_bytes(1, d) // 2, np.uint16) for d in plan.devices(1)}
        emulate_lowered(plan, sbufs, dbufs)
        for d in plan.devices(1):
            assert np.array_equal(dbufs[d], O.fill(m, dst, c, d, i)), (i, src, dst, d)
