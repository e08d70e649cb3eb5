"""CPU checks of the test infrastructure the full-size GPU parity relies on.

* The streamed oracle windows (orc_fill_range / orc_check_range) equal the
  whole-shard oracle fill on random windows, and the checker finds and
  locates a single flipped element.
* The special-value fill (seed bit 62): the product's value function (the
  __host__ __device__ code behind the GPU fill/verify kernels) and the
  oracle's agree with a third, pure-Python restatement written here, and the
  mode really produces every class of special bf16 word.
* Special-value shards survive the product's lowered rectangles applied on
  CPU, bit for bit.
"""
from __future__ import annotations

import dataclasses
import random

import numpy as np
import pytest

from _helpers import emulate_lowered, placement, random_placement
from oracle import oracle as O
from paper_2406_14088_b200 import rlplan as P
from paper_2406_14088_b200._lib import lib
from paper_2406_14088_b200.rlplan import BALANCED, SPEC

SPECIAL = O.SEED_SPECIAL
M64 = (1 << 64) - 1
TINY_GQA = dataclasses.replace(P.MODELS["tiny"], name="tiny_gqa", hidden_size=512, num_attention_heads=16,
                               num_kv_heads=8, intermediate_size=1024)


def py_value(seed: int, tensor: int, index: int) -> int:
    """Independent restatement of DESIGN.md §3 "Weights" (splitmix64 finaliser,
    then the normal or the special-value mapping)."""
    z = ((seed ^ (tensor << 40) ^ index) + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    z ^= z >> 31
    if not seed & SPECIAL:
        return ((z >> 63) << 15) | ((117 + ((z >> 8) & 7)) << 7) | (z & 0x7F)
    sign = 0x8000 if (z >> 16) & 1 else 0
    m = (z >> 17) & 0x7F
    return {0: sign, 1: sign | 0x7F80, 2: sign | 0x7FC0 | (m & 0x3F), 3: sign | 0x7F80 | (1 + m % 63),
            4: sign | m | 1, 5: sign | 0x7F7F, 6: sign | 0x0080}.get((z >> 24) & 15, z & 0xFFFF)


@pytest.mark.parametrize("seed", [0, 5, 2**63 + 7, SPECIAL, SPECIAL | 3, SPECIAL | (2**63 + 11)])
def test_value_function_three_way(seed):
    rng = random.Random(seed & 0xFFFF)
    for _ in range(3000):
        t, i = rng.randrange(1 << 12), rng.randrange(1 << 40)
        want = py_value(seed, t, i)
        assert O.value(seed, t, i) == want
        assert lib.rr_weight_value(seed, t, i) == want


def classify(v: np.ndarray) -> dict:
    exp, man = (v >> 7) & 0xFF, v & 0x7F
    return {
        "zero+": int(np.count_nonzero(v == 0)), "zero-": int(np.count_nonzero(v == 0x8000)),
        "inf": int(np.count_nonzero((exp == 0xFF) & (man == 0))),
        "qnan": int(np.count_nonzero((exp == 0xFF) & (man & 0x40 != 0))),
        "snan": int(np.count_nonzero((exp == 0xFF) & (man != 0) & (man & 0x40 == 0))),
        "denormal": int(np.count_nonzero((exp == 0) & (man != 0))),
        "max": int(np.count_nonzero((v & 0x7FFF) == 0x7F7F)),
        "min_normal": int(np.count_nonzero((v & 0x7FFF) == 0x0080)),
    }


def test_special_mode_covers_every_class():
    vals = np.array([O.value(SPECIAL | 9, t, i) for t in range(3) for i in range(20000)], dtype=np.uint16)
    counts = classify(vals)
    assert all(n > 100 for n in counts.values()), counts
    # NaN payloads vary (they must survive as distinct words)
    nans = vals[((vals >> 7) & 0xFF) == 0xFF]
    assert len(np.unique(nans)) > 100
    assert len(np.unique(vals)) > 20000  # arbitrary 16-bit patterns fill the rest


def test_windows_match_whole_shard_fill():
    rng = random.Random(7)
    c = P.b200_cluster(8)
    checked = 0
    for i in range(12):
        m = rng.choice([TINY_GQA, dataclasses.replace(TINY_GQA, name="tiny_mqa", num_attention_heads=8,
                                                      num_kv_heads=1, num_layers=3)])
        p = random_placement(rng, m)
        for d in range(8):
            n = O.shard_bytes(m, p, c, d)
            if not n:
                continue
            seed = rng.choice([3, SPECIAL | 3])
            full = O.fill(m, p, c, d, seed)
            assert np.array_equal(O.fill_mt(m, p, c, d, seed, threads=3), full)
            for _ in range(4):
                a = rng.randrange(0, n // 2) * 2
                b = rng.randrange(a // 2, n // 2 + 1) * 2
                w = np.empty((b - a) // 2, np.uint16)
                O.fill_range_into(m, p, c, d, seed, a, b - a, w.ctypes.data, threads=2)
                assert np.array_equal(w, full[a // 2:b // 2]), (i, d, a, b)
                assert O.check_range(m, p, c, d, seed, a, b - a, w.ctypes.data, threads=2) == (0, -1)
                if b > a:
                    k = rng.randrange(len(w))
                    w[k] ^= 0x8000
                    assert O.check_range(m, p, c, d, seed, a, b - a, w.ctypes.data, threads=2) == (1, k)
                checked += 1
    assert checked > 30


@pytest.mark.parametrize("sp,dp", [
    ((1, 1, 8, 0, 0), (1, 8, 1, 0, 0)),
    ((4, 1, 2, 2, 1), (1, 1, 8, 1, 1)),
    ((2, 1, 4, 0, 0), (1, 1, 8, 0, 0)),
    ((2, 1, 4, 0, 0), (1, 2, 4, 0, 0)),
])
@pytest.mark.parametrize("policy", [SPEC, BALANCED])
def test_special_values_through_lowered_rectangles(sp, dp, policy):
    c = P.b200_cluster(8)
    src = placement(8, *sp[:3], qkv=sp[3], gate_up=sp[4])
    dst = placement(8, *dp[:3], qkv=dp[3], gate_up=dp[4])
    plan = P.plan_param_realloc(TINY_GQA, src, dst, c, policy)
    seed = SPECIAL | 21
    sbufs = {d: O.fill(TINY_GQA, src, c, d, seed) for d in plan.devices(0)}
    dbufs = {d: np.zeros(plan.shard_bytes(1, d) // 2, np.uint16) for d in plan.devices(1)}
    emulate_lowered(plan, sbufs, dbufs)
    for d in plan.devices(1):
        assert np.array_equal(dbufs[d], O.fill(TINY_GQA, dst, c, d, seed)), f"device {d}"
