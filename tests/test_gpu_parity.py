"""GPU parity: the sm_100a reallocation kernels through the C ABI vs the CPU
oracle (bit-exact), on the same hash-initialised bf16 weights.

Small cases compare every destination byte with the oracle's expected shard
(oracle/realloc_oracle.c orc_fill) and with the oracle's CPU reallocation;
full-size BASELINE configs use size-independent properties (device-side
regenerate-and-compare of every shard, train->gen->train round trip,
sampled byte comparison against the oracle)."""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest

from _helpers import emulate_lowered, op_tuple, placement
from oracle import oracle as O
from paper_2406_14088_b200 import runtime as R
from paper_2406_14088_b200.rlplan import BALANCED, MODELS, SPEC, b200_cluster, plan_param_realloc
from paper_2406_14088_b200.workloads import WORKLOADS

pytestmark = pytest.mark.gpu

TINY_GQA = dataclasses.replace(MODELS["tiny"], name="tiny_gqa", hidden_size=512, num_attention_heads=16,
                               num_kv_heads=8, intermediate_size=1024)


def run_virtual(model, src, dst, cluster, policy=BALANCED, mode=R.PUSH, chunk=0, seed=11, kernel=0):
    plan = plan_param_realloc(model, src, dst, cluster, policy)
    vc = R.VirtualCluster(plan, 0)
    try:
        vc.fill_sources(seed)
        # the GPU fill is the oracle's value function, byte for byte
        for d, b in vc.src.items():
            assert np.array_equal(b.to_host(), O.fill(model, src, cluster, d, seed)), f"fill differs on {d}"
        ex = vc.executor(mode, chunk, kernel)
        ex.launch()
        R.stream_sync()
        got = {d: b.to_host() for d, b in vc.dst.items()}
        ex.close()
    finally:
        vc.free()
    return plan, got


def expected(model, src, dst, cluster, seed=11):
    return {d: O.fill(model, dst, cluster, d, seed) for d in dst.mesh.devices(cluster)}


def oracle_cpu_realloc(model, src, dst, cluster, policy, seed=11):
    ops, loc, _tb, _et = O.plan(model, src, dst, cluster, policy)
    n = cluster.device_count()
    sb = [O.fill(model, src, cluster, d, seed) if d in src.mesh.devices(cluster) else None for d in range(n)]
    db = [np.zeros(O.shard_bytes(model, dst, cluster, d) // 2, np.uint16) if d in dst.mesh.devices(cluster)
          else None for d in range(n)]
    O.execute(model, src, dst, cluster, ops + loc, sb, db, 4)
    return {d: db[d] for d in range(n) if db[d] is not None}


def assert_same(got, want):
    assert set(got) == set(want)
    for d in want:
        g, w = got[d], want[d]
        assert g.shape == w.shape, f"device {d}: shard size {g.shape} vs {w.shape}"
        bad = np.flatnonzero(g != w)
        assert bad.size == 0, f"device {d}: {bad.size} elements differ, first at {bad[0]}"


def test_tiny_baseline_config_bitexact(need_gpu):
    """BASELINE.json configs[0]: (pp1,dp1,tp2)->(pp1,dp2,tp1) on 2 devices."""
    w = WORKLOADS["tiny_tp2_to_dp2"]
    src, dst = w.phases[0]
    c = w.cluster()
    for policy in (SPEC, BALANCED):
        for mode in (R.PUSH, R.PULL):
            _plan, got = run_virtual(w.model, src, dst, c, policy, mode)
            assert_same(got, expected(w.model, src, dst, c))
            assert_same(got, oracle_cpu_realloc(w.model, src, dst, c, policy))


@pytest.mark.parametrize("model,sp,dp", [
    ("tiny", (1, 1, 2), (1, 2, 1)),        # BASELINE configs[0]: 3.4 MB, latency-bound
    ("tiny", (1, 1, 2), (2, 1, 1)),        # tp -> pp
    ("tiny", (1, 1, 4), (1, 4, 1)),        # 4-way all-gather, strided row-parallel rows
    ("tiny_gqa", (2, 1, 2), (1, 1, 4)),    # pp + tp remap, k/v split
])
def test_small_phase_recut_bitexact(need_gpu, model, sp, dp):
    """With the default chunk, a phase below the small-phase size is re-cut to
    about one item per resident CTA (capi_exec.cpp refine_small); every byte
    still lands exactly once and in place."""
    m = MODELS["tiny"] if model == "tiny" else TINY_GQA
    n = sp[0] * sp[1] * sp[2]
    c = b200_cluster(max(n, 2))
    src, dst = placement(n, *sp), placement(n, *dp)
    plan = plan_param_realloc(m, src, dst, c, BALANCED)
    vc = R.VirtualCluster(plan, 0)
    try:
        vc.fill_sources(3)
        coarse = vc.executor(R.PUSH, 256 << 10, None)  # explicit chunk: no re-cut
        fine = vc.executor(R.PUSH, 0, None)
        assert fine.items > coarse.items, (fine.items, coarse.items)
        assert fine.bytes_written == coarse.bytes_written and fine.bytes_read == coarse.bytes_read
        fine.launch()
        R.stream_sync()
        got = {d: b.to_host() for d, b in vc.dst.items()}
        coarse.close()
        fine.close()
    finally:
        vc.free()
    assert_same(got, expected(m, src, dst, c, seed=3))


@pytest.mark.parametrize("sp,dp", [
    ((4, 1, 2, 2, 1), (1, 1, 8, 1, 1)),   # 34B-style: pp4 tp2 Megatron-grouped -> tp8 concat
    ((2, 1, 4, 2, 1), (1, 2, 4, 0, 0)),   # pipeline remap + fused -> separate
    ((1, 2, 4, 1, 0), (2, 1, 4, 2, 1)),   # dp2 concat -> pp2 grouped
    ((1, 8, 1, 2, 1), (4, 1, 2, 0, 0)),   # dp8 replicas -> pp4 tp2
    ((1, 1, 8, 0, 0), (1, 8, 1, 0, 0)),   # 7B-style tp8 -> dp8 all-gather
    ((2, 1, 4, 0, 0), (1, 1, 8, 0, 0)),   # 70B-style pp2 tp4 -> tp8
])
@pytest.mark.parametrize("mode", [R.PUSH, R.PULL])
@pytest.mark.parametrize("kernel", [0, 1, 5])
def test_reinterleave_bitexact(need_gpu, sp, dp, mode, kernel):
    c = b200_cluster(8)
    src = placement(8, *sp[:3], qkv=sp[3], gate_up=sp[4])
    dst = placement(8, *dp[:3], qkv=dp[3], gate_up=dp[4])
    # a small chunk forces row- and column-splitting of the copy items
    _plan, got = run_virtual(TINY_GQA, src, dst, c, BALANCED, mode, chunk=4096, kernel=kernel)
    assert_same(got, expected(TINY_GQA, src, dst, c))


@pytest.mark.parametrize("sp,dp", [
    ((1, 1, 8, 0, 0), (1, 8, 1, 0, 0)),   # all-gather, strided row-parallel pieces
    ((4, 1, 2, 2, 1), (1, 1, 8, 1, 1)),   # grouped -> concat reinterleave
    ((2, 1, 4, 0, 0), (1, 2, 4, 0, 0)),   # stage remap
    ((1, 8, 1, 0, 0), (1, 1, 8, 0, 0)),   # local slicing
])
@pytest.mark.parametrize("mode", [R.PUSH, R.PULL])
@pytest.mark.parametrize("kernel", [0, 1, 5])
def test_special_value_words_survive_every_kernel(need_gpu, sp, dp, mode, kernel):
    """Signed zeros, infinities, quiet and signalling NaNs with payloads,
    subnormals, extreme normals and arbitrary 16-bit words are moved as
    opaque bytes by the LDG/STG kernel and both TMA bulk rings,
    push and pull, whole items and 4 KiB split items."""
    c = b200_cluster(8)
    src = placement(8, *sp[:3], qkv=sp[3], gate_up=sp[4])
    dst = placement(8, *dp[:3], qkv=dp[3], gate_up=dp[4])
    for chunk in (0, 4096):
        seed = O.SEED_SPECIAL | (40 + chunk % 7)
        _plan, got = run_virtual(TINY_GQA, src, dst, c, BALANCED, mode, chunk=chunk, kernel=kernel, seed=seed)
        assert_same(got, expected(TINY_GQA, src, dst, c, seed=seed))


def test_special_value_words_2byte_path(need_gpu):
    """The 2-byte element path (SPEC.md:47 tiny spec, 8-byte rows)."""
    m = MODELS["spec_tiny"]
    c = b200_cluster(2)
    src, dst = placement(2, 1, 1, 2), placement(2, 1, 2, 1)
    seed = O.SEED_SPECIAL | 3
    _plan, got = run_virtual(m, src, dst, c, SPEC, seed=seed, kernel=1)
    assert_same(got, expected(m, src, dst, c, seed=seed))


@pytest.mark.parametrize("kernel", [0, 1])
def test_spec_tiny_unaligned_elements(need_gpu, kernel):
    """SPEC.md:47 tiny spec (h=4): 8-byte rows take the 2-byte element path."""
    m = MODELS["spec_tiny"]
    c = b200_cluster(2)
    src = placement(2, 1, 2, 1)
    dst = placement(2, 1, 1, 2)
    _plan, got = run_virtual(m, src, dst, c, SPEC, kernel=kernel)
    assert_same(got, expected(m, src, dst, c))


def test_disjoint_meshes_bitexact(need_gpu):
    """Parameter sync between disjoint meshes: dp4 on GPUs 0-3 -> tp4 on 4-7."""
    c = b200_cluster(8)
    src = placement(4, 1, 4, 1, offset=0)
    dst = placement(4, 1, 1, 4, offset=4)
    for kernel in (0, 5):
        _plan, got = run_virtual(TINY_GQA, src, dst, c, BALANCED, kernel=kernel)
        assert_same(got, expected(TINY_GQA, src, dst, c))


def test_7b_train_gen_roundtrip_full_size(need_gpu):
    """BASELINE.json configs[1] at full size on one GPU (8 plan devices):
    every generation shard verified on device, then gen->train reproduces the
    original training shards exactly (round trip), one shard compared byte
    for byte with the oracle."""
    w = WORKLOADS["llama7b_tp8_dp8_roundtrip"]
    c = w.cluster()
    plans = [plan_param_realloc(w.model, s, d, c, BALANCED) for (s, d) in w.phases]
    rr = R.RankRealloc(plans, {"train": (0, R.SRC), "gen": (0, R.DST)}, [("train", "gen"), ("gen", "train")],
                       rank=0, world=1, cuda_device=0)
    try:
        seed = 3
        for d, b in rr.buffers["train"].items():
            R.fill_shard(plans[0], R.SRC, d, b.ptr, seed)
        want3 = rr.buffers["train"][3].to_host()
        assert np.array_equal(want3, O.fill(w.model, w.phases[0][0], c, 3, seed))
        rr.run_phase(0)
        R.stream_sync()
        for d, b in rr.buffers["gen"].items():
            assert R.verify_shard(plans[0], R.DST, d, b.ptr, seed) == (0, -1), f"gen shard {d}"
        # wipe the training shards, then rebuild them from the generation replicas
        for b in rr.buffers["train"].values():
            b.zero()
        rr.run_phase(1)
        R.stream_sync()
        for d, b in rr.buffers["train"].items():
            assert R.verify_shard(plans[1], R.DST, d, b.ptr, seed) == (0, -1), f"train shard {d}"
        assert np.array_equal(rr.buffers["train"][3].to_host(), want3)
    finally:
        rr.close()


def test_random_placement_pairs_bitexact_on_gpu(need_gpu):
    """Fuzz: 80 random (src, dst) placement pairs (sub-meshes, pp/dp/tp,
    Separate/Concat/Grouped layouts, both policies, push and pull, both copy
    kernels, random work-item sizes) through the sm_100a kernels, each
    bit-exact against the oracle's expected destination shards."""
    import random

    from _helpers import random_placement
    rng = random.Random(14088)
    c = b200_cluster(8)
    models = [TINY_GQA, dataclasses.replace(TINY_GQA, num_layers=5, has_output_head=False),
              dataclasses.replace(MODELS["tiny"], num_layers=3),
              # 1 and 2 KV heads: replicated-head layouts (G6) at tp > kv
              dataclasses.replace(TINY_GQA, name="tiny_mqa", num_attention_heads=8, num_kv_heads=1, num_layers=3),
              dataclasses.replace(TINY_GQA, name="tiny_kv2", num_attention_heads=8, num_kv_heads=2, num_layers=2)]
    for i in range(80):
        m = rng.choice(models)
        src, dst = random_placement(rng, m), random_placement(rng, m)
        policy = rng.choice([SPEC, BALANCED])
        mode = rng.choice([R.PUSH, R.PULL])
        kernel = rng.choice([0, 1, 5])
        chunk = rng.choice([0, 4096, 65536])
        _plan, got = run_virtual(m, src, dst, c, policy, mode, chunk=chunk, seed=100 + i, kernel=kernel)
        assert_same(got, expected(m, src, dst, c, seed=100 + i))
