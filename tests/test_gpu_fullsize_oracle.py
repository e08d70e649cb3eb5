"""Full-size byte parity against the oracle (replaying
the ops reproduces exactly the destination requirement).

Every BASELINE.json config at its full shapes runs through the sm_100a
kernels on one GPU (all plan devices co-resident), and EVERY byte of every
destination shard is compared with the oracle's expected shard, streamed
window by window (orc_check_range, oracle/realloc_oracle.c): no check goes
through the product's own layout tables or verify kernel. The 70B config
does not fit one GPU whole (282 GB of shards), so its destinations are
checked a few at a time at full size, each time with exactly the source
shards their ops read. Seeds alternate between the normal and the
special-value fill (signed zeros, infinities, NaN payloads, subnormals,
arbitrary 16-bit words)."""
from __future__ import annotations

import time

import pytest

from _helpers import oracle_compare_device
from oracle import oracle as O
from paper_2406_14088_b200 import runtime as R
from paper_2406_14088_b200.rlplan import BALANCED, SPEC, plan_param_realloc
from paper_2406_14088_b200.workloads import WORKLOADS

pytestmark = pytest.mark.gpu

SPECIAL = O.SEED_SPECIAL


@pytest.fixture(scope="module")
def hosts():
    bufs = [R.HostBuffer(256 << 20), R.HostBuffer(256 << 20)]
    yield bufs
    for b in bufs:
        b.free()


def _check_all(model, placement, cluster, seed, bufs, hosts, what):
    t0 = time.time()
    total = 0
    for d, b in sorted(bufs.items()):
        bad, first = oracle_compare_device(model, placement, cluster, d, seed, b.ptr, b.nbytes, hosts=hosts)
        assert bad == 0, f"{what}: device {d} differs from the oracle in {bad} elements (first at byte {first})"
        total += b.nbytes
    print(f"{what}: {total / 1e9:.2f} GB compared with the oracle in {time.time() - t0:.1f} s")
    return total


def test_7b_roundtrip_every_byte_special_values(need_gpu, hosts):
    """configs[1] LLaMA-7B (pp1,dp1,tp8) -> (pp1,dp8,tp1) -> back, special-value
    weights: the 8 generation replicas (128.5 GB) and the rebuilt training
    shards are compared byte for byte with the oracle."""
    w = WORKLOADS["llama7b_tp8_dp8_roundtrip"]
    c = w.cluster()
    (train, gen), _ = w.phases
    plans = [plan_param_realloc(w.model, s, d, c, BALANCED) for (s, d) in w.phases]
    rr = R.RankRealloc(plans, {"train": (0, R.SRC), "gen": (0, R.DST)}, [("train", "gen"), ("gen", "train")],
                       rank=0, world=1, cuda_device=0)
    try:
        seed = SPECIAL | 4
        for d, b in rr.buffers["train"].items():
            R.fill_shard(plans[0], R.SRC, d, b.ptr, seed)
        R.stream_sync()
        _check_all(w.model, train, c, seed, rr.buffers["train"], hosts, "7B train shards (GPU fill)")
        rr.run_phase(0)
        R.stream_sync()
        _check_all(w.model, gen, c, seed, rr.buffers["gen"], hosts, "7B gen replicas")
        for b in rr.buffers["train"].values():
            b.zero()
        rr.run_phase(1)
        R.stream_sync()
        _check_all(w.model, train, c, seed, rr.buffers["train"], hosts, "7B train shards rebuilt")
    finally:
        rr.close()


@pytest.mark.parametrize("name,seed", [("llama13b_pp2tp4_to_dp2tp4", 6),
                                       ("llama34b_critic_pp4tp2_to_tp8", SPECIAL | 7)])
def test_full_config_every_byte(need_gpu, hosts, name, seed):
    """configs[2] 13B pipeline-stage remap (84 GB of shards) and configs[3]
    34B critic fused-QKV/gate-up reinterleave (137 GB), whole."""
    w = WORKLOADS[name]
    c = w.cluster()
    (src, dst), = w.phases
    plan = plan_param_realloc(w.model, src, dst, c, BALANCED)
    vc = R.VirtualCluster(plan, 0)
    try:
        vc.fill_sources(seed)
        ex = vc.executor(R.PUSH)
        ex.launch()
        R.stream_sync()
        n = _check_all(w.model, dst, c, seed, vc.dst, hosts, name)
        assert n == sum(plan.shard_bytes(R.DST, d) for d in plan.devices(R.DST))
        ex.close()
    finally:
        vc.free()


def _sources_read(plan, dsts):
    return sorted({s for s, ds, _r in plan.lowered() if set(ds) & set(dsts)})


@pytest.mark.parametrize("policy", [BALANCED, SPEC])
def test_70b_full_size_every_byte(need_gpu, hosts, policy):
    """configs[4] LLaMA-70B (pp2,dp1,tp4) -> (pp1,dp1,tp8) at full size
    (17.6 GB shards, vocab slices of 250 MB, item offsets far beyond 2^32).
    Destinations are taken in groups that fit the GPU together with exactly
    the sources their ops read; a pull executor driving the group fills them;
    every byte is compared with the oracle."""
    import torch
    w = WORKLOADS["llama70b_pp2tp4_to_tp8"]
    c = w.cluster()
    (src, dst), = w.phases
    plan = plan_param_realloc(w.model, src, dst, c, policy)
    free = torch.cuda.mem_get_info(0)[0]
    seed = 8 if policy == BALANCED else SPECIAL | 8
    todo = plan.devices(R.DST)
    checked = 0
    while todo:
        group = [todo[0]]
        for d in todo[1:]:
            g = group + [d]
            need = sum(plan.shard_bytes(R.SRC, s) for s in _sources_read(plan, g)) + \
                sum(plan.shard_bytes(R.DST, x) for x in g)
            if need < 0.85 * free:
                group = g
        todo = [d for d in todo if d not in group]
        srcs = _sources_read(plan, group)
        sbufs = {s: R.DeviceBuffer(0, plan.shard_bytes(R.SRC, s)) for s in srcs}
        dbufs = {d: R.DeviceBuffer(0, plan.shard_bytes(R.DST, d)) for d in group}
        try:
            for d, b in dbufs.items():
                b.zero()
            for s, b in sbufs.items():
                R.fill_shard(plan, R.SRC, s, b.ptr, seed)
            ex = R.Executor(plan, 0, {s: b.ptr for s, b in sbufs.items()}, {d: b.ptr for d, b in dbufs.items()},
                            group, R.PULL)
            ex.launch()
            R.stream_sync()
            ex.close()
            checked += _check_all(w.model, dst, c, seed, dbufs, hosts, f"70B destinations {group} (sources {srcs})")
        finally:
            for b in list(sbufs.values()) + list(dbufs.values()):
                b.free()
    assert checked == sum(plan.shard_bytes(R.DST, d) for d in plan.devices(R.DST))
