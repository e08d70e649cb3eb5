"""Onload of parked parameters pipelined with the reallocation (
SURVEY.md §8(f) rank 2): source shards come from pinned host memory in
chunks on a side stream, copy segments start as their chunk lands. Results
are bit-exact against the CPU oracle."""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest

from _helpers import placement
from oracle import oracle as O
from paper_2406_14088_b200 import runtime as R
from paper_2406_14088_b200.rlplan import BALANCED, MODELS, b200_cluster, plan_param_realloc

pytestmark = pytest.mark.gpu

TINY_GQA = dataclasses.replace(MODELS["tiny"], name="tiny_gqa", hidden_size=512, num_attention_heads=16,
                               num_kv_heads=8, intermediate_size=1024)


@pytest.mark.parametrize("sp,dp", [((1, 1, 8, 0, 0), (1, 8, 1, 0, 0)), ((4, 1, 2, 2, 1), (1, 1, 8, 1, 1))])
@pytest.mark.parametrize("kernel", [0, 1])
@pytest.mark.parametrize("seed", [31, O.SEED_SPECIAL | 31])
def test_onload_pipeline_bitexact(need_gpu, sp, dp, kernel, seed):
    import torch
    c = b200_cluster(8)
    src = placement(8, *sp[:3], qkv=sp[3], gate_up=sp[4])
    dst = placement(8, *dp[:3], qkv=dp[3], gate_up=dp[4])
    plan = plan_param_realloc(TINY_GQA, src, dst, c, BALANCED)
    vc = R.VirtualCluster(plan, 0)
    hosts = {}
    try:
        for d, b in vc.src.items():   # parked parameters: pinned host copies of the source shards
            hb = R.HostBuffer(b.nbytes)
            hb.array()[:] = O.fill(TINY_GQA, src, c, d, seed)
            hosts[d] = hb
            b.zero()
        ex = vc.executor(R.PUSH, 4096, kernel)
        ex.enable_onload({d: b.nbytes for d, b in vc.src.items()}, chunk_bytes=64 << 10)
        copy = torch.cuda.Stream()
        for _ in range(2):  # re-launchable
            for b in vc.dst.values():
                b.zero()
            ex.launch_onload({d: h.ptr for d, h in hosts.items()}, copy, torch.cuda.current_stream())
            torch.cuda.synchronize()
            for d, b in vc.dst.items():
                assert np.array_equal(b.to_host(), O.fill(TINY_GQA, dst, c, d, seed)), d
        ex.close()
    finally:
        vc.free()
        for h in hosts.values():
            h.free()


@pytest.mark.parametrize("kernel", [0, 1])
@pytest.mark.parametrize("seed", [17, O.SEED_SPECIAL | 17])
def test_offload_overlaps_reallocation_then_onload_round_trip(need_gpu, kernel, seed):
    """Park the source shards in pinned host memory while the reallocation
    reads them ("host-device (e.g., offload)"), wipe them,
    then onload them back pipelined with the same reallocation: every host
    copy and every destination shard is bit-exact."""
    import torch
    c = b200_cluster(8)
    src = placement(8, 1, 1, 8)
    dst = placement(8, 1, 8, 1)
    plan = plan_param_realloc(TINY_GQA, src, dst, c, BALANCED)
    vc = R.VirtualCluster(plan, 0)
    hosts = {}
    try:
        vc.fill_sources(seed=seed)
        for d, b in vc.src.items():
            hosts[d] = R.HostBuffer(b.nbytes)
            hosts[d].array()[:] = 0
        ex = vc.executor(R.PUSH, 8192, kernel)
        copy = torch.cuda.Stream()
        cur = torch.cuda.current_stream()
        ex.launch_offload({d: b.nbytes for d, b in vc.src.items()}, {d: h.ptr for d, h in hosts.items()}, copy, cur)
        ex.launch(cur)
        torch.cuda.synchronize()
        for d, h in hosts.items():
            assert np.array_equal(h.array(), O.fill(TINY_GQA, src, c, d, seed)), d
        for d, b in vc.dst.items():
            assert np.array_equal(b.to_host(), O.fill(TINY_GQA, dst, c, d, seed)), d
        for b in list(vc.src.values()) + list(vc.dst.values()):
            b.zero()
        ex.enable_onload({d: b.nbytes for d, b in vc.src.items()}, chunk_bytes=32 << 10)
        ex.launch_onload({d: h.ptr for d, h in hosts.items()}, copy, cur)
        torch.cuda.synchronize()
        for d, b in vc.dst.items():
            assert np.array_equal(b.to_host(), O.fill(TINY_GQA, dst, c, d, seed)), d
        ex.close()
    finally:
        vc.free()
        for h in hosts.values():
            h.free()
