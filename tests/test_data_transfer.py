"""plan_data_transfer: product vs the oracle's C
restatement, the SPEC examples, the replay oracle on random pairs, and the
product's lowering applied on CPU vs the oracle's expected consumer data.
The GPU test runs the same plans through the sm_100a kernels."""
from __future__ import annotations

import random

import numpy as np
import pytest

from _helpers import op_tuple
from oracle import oracle as O
from paper_2406_14088_b200 import rlplan as P
from paper_2406_14088_b200.rlplan import BALANCED, SPEC


def pl(gpus, pp, dp, tp, offset=0):
    return P.Placement(P.DeviceMesh(0, 1, offset, gpus), P.ParallelStrategy(dp=dp, tp=tp, pp=pp))


def both(prod, cons, c, per_shard, policy):
    p = P.plan_data_transfer(prod, cons, per_shard, c, policy)
    o = O.plan_data(prod, cons, c, per_shard, policy)
    assert o is not None
    ops, loc, tb, et = o
    assert [op_tuple(x) for x in p.ops] == ops
    assert [op_tuple(x) for x in p.local_ops] == loc
    assert p.total_bytes == tb
    assert p.est_time == pytest.approx(et, rel=1e-12)
    return p, ops, loc


def emulate(plan, prod, cons, c, total, seed):
    n = c.device_count()
    src = {d: O.data_fill(prod, c, d, True, total, seed) for d in range(n)
           if O.data_shard_bytes(prod, c, d, True, total)}
    dst = {d: np.zeros(plan.shard_bytes(1, d) // 2, np.uint16) for d in cons.mesh.devices(c)}
    for s, dsts, rects in plan.lowered():
        for d in dsts:
            for (so, do, rb, _sp, _dp, rows) in rects:
                assert rows == 1
                dst[d].view(np.uint8)[do:do + rb] = src[s].view(np.uint8)[so:so + rb]
    return dst


def test_identical_placements_empty_plan():
    """SPEC.md:584."""
    c = P.b200_cluster(8)
    for p in (pl(8, 2, 2, 2), pl(4, 1, 4, 1), pl(2, 1, 1, 2)):
        plan, ops, _ = both(p, p, c, 1 << 16, SPEC)
        assert plan.ops == [] and plan.total_bytes == 0


def test_dp2_to_dp1_consumer_gathers_both_shards():
    """producer dp=2 -> consumer dp=1 on a superset mesh: each
    consumer device gathers both shards; bytes = total minus what it holds."""
    c = P.b200_cluster(8)
    prod = pl(2, 1, 2, 1)
    cons = pl(4, 1, 1, 4)      # superset mesh gpu[0-3]
    per = 1 << 20
    plan, ops, loc = both(prod, cons, c, per, SPEC)
    total = 2 * per
    recv = {d: 0 for d in range(4)}
    for op in plan.ops:
        for d in op.dst:
            recv[d] += op.bytes
    assert recv[0] == total - per and recv[1] == total - per   # hold one shard each
    assert recv[2] == total and recv[3] == total                # hold nothing
    assert O.replay_data(prod, cons, c, per, ops, loc) is None


def _random_data_placement(rng, gpus=8):
    size = rng.choice([1, 2, 4, 8])
    off = rng.randrange(0, gpus // size) * size
    dims = [(dp, tp, size // (dp * tp)) for dp in (1, 2, 4, 8) for tp in (1, 2, 4, 8)
            if size % (dp * tp) == 0]
    dp, tp, pp = rng.choice(dims)
    return pl(size, pp, dp, tp, off)


def test_random_pairs_replay_and_bytes():
    rng = random.Random(578)
    c = P.b200_cluster(8)
    for _ in range(300):
        prod, cons = _random_data_placement(rng), _random_data_placement(rng)
        per = 4096 * rng.choice([1, 3, 8])
        policy = rng.choice([SPEC, BALANCED])
        plan, ops, loc = both(prod, cons, c, per, policy)
        assert O.replay_data(prod, cons, c, per, ops, loc) is None
        total = per * prod.strategy.dp
        got = emulate(plan, prod, cons, c, total, 5)
        for d in cons.mesh.devices(c):
            want = O.data_fill(cons, c, d, False, total, 5)
            assert np.array_equal(got[d], want), (prod, cons, d)


def test_invalid_data_plans():
    c = P.b200_cluster(8)
    with pytest.raises(P.ValidationError, match="dp\\*tp\\*pp must equal the mesh size"):
        P.plan_data_transfer(pl(4, 1, 2, 1), pl(4, 1, 4, 1), 4096, c)
    with pytest.raises(P.ValidationError, match="equal bf16 slices"):
        P.plan_data_transfer(pl(4, 1, 4, 1), pl(8, 1, 8, 1), 6, c)   # 24 bytes over lcm 8
    assert O.plan_data(pl(4, 1, 2, 1), pl(4, 1, 4, 1), c, 4096) is None


@pytest.mark.gpu
def test_data_transfer_on_gpu(need_gpu):
    from paper_2406_14088_b200 import runtime as R
    c = P.b200_cluster(8)
    for prod, cons in [(pl(4, 2, 2, 1), pl(8, 1, 4, 2)), (pl(8, 1, 8, 1), pl(2, 1, 1, 2, 6)),
                       (pl(2, 1, 2, 1), pl(4, 1, 1, 4))]:
        per = 1 << 18
        plan = P.plan_data_transfer(prod, cons, per, c, BALANCED)
        vc = R.VirtualCluster(plan, 0)
        try:
            for d, b in vc.src.items():
                R.fill_shard(plan, R.SRC, d, b.ptr, 13)
            ex = vc.executor()
            ex.launch()
            R.stream_sync()
            total = per * prod.strategy.dp
            for d, b in vc.dst.items():
                assert np.array_equal(b.to_host(), O.data_fill(cons, c, d, False, total, 13)), (prod, cons, d)
            ex.close()
        finally:
            vc.free()


def test_data_workloads_plan_and_cpu_sample():
    """The bench's data workloads build product plans that match the oracle,
    and the CPU arm's sample reproduces the consumer data."""
    import dataclasses
    import importlib.util
    import os
    from paper_2406_14088_b200.workloads import WORKLOADS
    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for name in ("data_gen_dp8_to_train_tp8", "data_gen_dp8_to_pp2dp2tp2"):
        w = dataclasses.replace(WORKLOADS[name], data_bytes=1 << 20)
        (prod, cons), = w.phases
        p, ops, loc = both(prod, cons, w.cluster(), w.data_bytes, BALANCED)
        assert [op_tuple(x) for x in w.plans(BALANCED)[0].ops] == ops
        pw = bench.plain_workload(name)  # the reference arm's own, product-free view of the workload
        pw.data_bytes = 1 << 20
        r = bench.cpu_realloc(pw, 1, 0, 1)
        assert r["correct"] and r["delivered"] == sum(b * len(d) for (_s, d, _p, b) in ops + loc) > 0


def test_reference_arm_workloads_match_product():
    """bench.py's reference arm builds every named workload from
    workloads.json without the product; the oracle plans it identically to
    the product's workload objects, and the `config` blocks of both arms
    agree."""
    import importlib.util
    import os
    from oracle import oracle as O
    from paper_2406_14088_b200.workloads import WORKLOADS
    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for name, w in WORKLOADS.items():
        pw = bench.plain_workload(name)
        assert bench.workload_config(pw) == bench.workload_config(w)
        assert len(pw.phases) == len(w.phases) and pw.devices == w.devices
        for (ps, pd), (s, d) in zip(pw.phases, w.phases):
            if w.data_bytes:
                assert O.plan_data(ps, pd, pw.cluster, w.data_bytes, 1) == O.plan_data(s, d, w.cluster(), w.data_bytes, 1)
            else:
                assert O.plan(pw.model, ps, pd, pw.cluster, 1) == O.plan(w.model, s, d, w.cluster(), 1)


def test_reference_arm_never_loads_the_product():
    """`bench.py --impl reference` runs the oracle's CPU reallocation on
    product-free workload objects: the process never maps librrealloc.so
    nor imports the package (the old reference arm did)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--workload', 'tiny_tp2_to_dp2', "
            "'--steps', '2', '--warmup', '1']; runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "print('PRODUCT' if 'librrealloc' in maps or any(m.startswith('paper_2406_14088_b200') "
            "for m in sys.modules) else 'CLEAN')")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    assert lines[-1] == "CLEAN", r.stdout
    import json
    line = json.loads(lines[-2])
    assert line["impl"] == "reference" and line["verified"] and line["cpu_baseline"]["kind"] == "port"
