"""Shared test helpers: placements for the BASELINE configs, op conversion,
and a numpy emulation of the product's lowered copy rectangles."""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Tuple

import numpy as np

from paper_2406_14088_b200.rlplan import (MODELS, DeviceMesh, ParallelStrategy, Placement, b200_cluster)


def mesh(gpus: int, offset: int = 0) -> DeviceMesh:
    return DeviceMesh(0, 1, offset, gpus)


def placement(gpus: int, pp: int, dp: int, tp: int, offset: int = 0, qkv: int = 0, gate_up: int = 0) -> Placement:
    """(pp, dp, tp) order as written in BASELINE.json configs."""
    return Placement(mesh(gpus, offset), ParallelStrategy(dp=dp, tp=tp, pp=pp), qkv, gate_up)


def op_tuple(op) -> tuple:
    p = op.payload
    return (op.src, tuple(op.dst), (p.layer_start, p.layer_end, p.tp_rank, p.tp_degree, p.replicated, p.part),
            op.bytes)


def scaled(name: str, layers: Optional[int] = None, vocab: Optional[int] = None):
    m = MODELS[name]
    kw = {}
    if layers is not None:
        kw["num_layers"] = layers
    if vocab is not None:
        kw["vocab_size"] = vocab
    return dataclasses.replace(m, **kw) if kw else m


# BASELINE.json configs (pp, dp, tp) -> (pp, dp, tp), with layouts.
BASELINE_CONFIGS = {
    "tiny_tp2_to_dp2": ("tiny", 2, (1, 1, 2, 0, 0), (1, 2, 1, 0, 0)),
    "7b_tp8_to_dp8": ("llama7b", 8, (1, 1, 8, 0, 0), (1, 8, 1, 0, 0)),
    "7b_dp8_to_tp8": ("llama7b", 8, (1, 8, 1, 0, 0), (1, 1, 8, 0, 0)),
    "13b_pp2tp4_to_dp2tp4": ("llama13b", 8, (2, 1, 4, 0, 0), (1, 2, 4, 0, 0)),
    "34b_pp4tp2_to_tp8_fused": ("llama34b_critic", 8, (4, 1, 2, 2, 1), (1, 1, 8, 1, 1)),
    "70b_pp2tp4_to_tp8": ("llama70b", 8, (2, 1, 4, 0, 0), (1, 1, 8, 0, 0)),
}


def config_placements(key: str):
    name, gpus, s, d = BASELINE_CONFIGS[key]
    src = placement(gpus, s[0], s[1], s[2], qkv=s[3], gate_up=s[4])
    dst = placement(gpus, d[0], d[1], d[2], qkv=d[3], gate_up=d[4])
    return MODELS[name], src, dst, b200_cluster(gpus)


def emulate_lowered(plan, src_bufs: Dict[int, np.ndarray], dst_bufs: Dict[int, np.ndarray]) -> None:
    """Apply the product's lowered rectangles with numpy (uint8 views)."""
    for s, dsts, rects in plan.lowered():
        sb = src_bufs[s].view(np.uint8)
        for d in dsts:
            db = dst_bufs[d].view(np.uint8)
            for (so, do, rb, sp, dp, rows) in rects:
                for r in range(rows):
                    db[do + r * dp: do + r * dp + rb] = sb[so + r * sp: so + r * sp + rb]


def random_placement(rng, model, gpus_per_node: int = 8) -> Placement:
    """A random valid placement on an aligned sub-mesh of one node: random
    size, offset, (pp, dp, tp), fused layouts and K/V layout (plan-parity and
    GPU fuzz)."""
    from paper_2406_14088_b200 import rlplan as P
    size = rng.choice([1, 2, 4, 8])
    offset = rng.randrange(0, gpus_per_node // size) * size
    while True:
        tp = rng.choice([t for t in (1, 2, 4, 8) if size % t == 0])
        pp = rng.choice([q for q in range(1, size // tp + 1) if (size // tp) % q == 0 and q <= model.num_layers])
        dp = size // (tp * pp)
        qkv = rng.choice([0, 1, 2])
        gu = rng.choice([0, 1])
        kv = rng.choice([0, 1])
        p = P.Placement(P.DeviceMesh(0, 1, offset, size), P.ParallelStrategy(dp=dp, tp=tp, pp=pp), qkv, gu, kv)
        try:
            P.validate_placement(model, p, P.b200_cluster(gpus_per_node))
            return p
        except P.ValidationError:
            continue


def oracle_compare_device(model, placement, cluster, dev: int, seed: int, dev_ptr: int, nbytes: int,
                          window: int = 256 << 20, hosts=None):
    """Compare every byte of a device-resident shard with the oracle's
    expected shard, window by window (orc_check_range, all host threads):
    window k + 1 is copied device->host while the oracle checks window k.
    Returns (mismatching bf16 elements, byte offset of the first one or -1).
    `hosts`: two reusable pinned buffers of >= window bytes (else allocated)."""
    from oracle import oracle as O
    from paper_2406_14088_b200 import runtime as R
    own = hosts is None
    if own:
        hosts = [R.HostBuffer(window), R.HostBuffer(window)]
    try:
        offs = list(range(0, nbytes, window))
        bad, first = 0, -1
        if offs:
            R.memcpy_async(hosts[0].ptr, dev_ptr, min(window, nbytes), 1)
        for k, off in enumerate(offs):
            R.stream_sync()
            n = min(window, nbytes - off)
            if k + 1 < len(offs):
                nxt = offs[k + 1]
                R.memcpy_async(hosts[(k + 1) % 2].ptr, dev_ptr + nxt, min(window, nbytes - nxt), 1)
            b, f = O.check_range(model, placement, cluster, dev, seed, off, n, hosts[k % 2].ptr)
            if b and first < 0:
                first = off + 2 * f
            bad += b
        R.stream_sync()
        return bad, first
    finally:
        if own:
            for h in hosts:
                h.free()
