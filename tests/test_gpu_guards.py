"""Out-of-bounds detection without compute-sanitizer (closed on the GPU pool):
every shard is surrounded by guard bytes with a known pattern; after the
reallocation kernels run (all copy engines, push and pull, 2-byte and
16-byte paths) the guards must be intact and the shards bit-exact."""
from __future__ import annotations

import ctypes
import dataclasses

import numpy as np
import pytest

from _helpers import placement
from oracle import oracle as O
from paper_2406_14088_b200 import runtime as R
from paper_2406_14088_b200._lib import check, lib
from paper_2406_14088_b200.rlplan import BALANCED, MODELS, SPEC, b200_cluster, plan_param_realloc

pytestmark = pytest.mark.gpu
GUARD = 64 << 10

TINY_GQA = dataclasses.replace(MODELS["tiny"], name="tiny_gqa", hidden_size=512, num_attention_heads=16,
                               num_kv_heads=8, intermediate_size=1024)


class Guarded:
    """A shard with GUARD bytes of 0xA5 before and after it."""

    def __init__(self, nbytes: int):
        self.nbytes = nbytes
        self.buf = R.DeviceBuffer(0, nbytes + 2 * GUARD)
        pattern = np.full((nbytes + 2 * GUARD) // 2 + 1, 0xA5A5, dtype=np.uint16)
        check(lib.rr_memcpy(self.buf.ptr, pattern.ctypes.data, nbytes + 2 * GUARD, 0, None, 1))
        check(lib.rr_memset(self.buf.ptr + GUARD, 0, nbytes, None))
        self.ptr = self.buf.ptr + GUARD

    def read(self):
        out = np.empty((self.nbytes + 2 * GUARD) // 2, dtype=np.uint16)
        check(lib.rr_memcpy(out.ctypes.data, self.buf.ptr, self.nbytes + 2 * GUARD, 1, None, 1))
        return out[: GUARD // 2], out[GUARD // 2: (GUARD + self.nbytes) // 2], out[(GUARD + self.nbytes) // 2:]


@pytest.mark.parametrize("model,sp,dp,gpus", [
    (TINY_GQA, (4, 1, 2, 2, 1), (1, 1, 8, 1, 1), 8),
    (TINY_GQA, (1, 8, 1, 2, 1), (4, 1, 2, 0, 0), 8),
    (MODELS["spec_tiny"], (1, 2, 1, 0, 0), (1, 1, 2, 0, 0), 2),   # 2-byte element path
])
@pytest.mark.parametrize("mode,kernel", [(R.PUSH, 0), (R.PUSH, 1), (R.PULL, 1), (R.PUSH, 5)])
def test_guards_intact(need_gpu, model, sp, dp, gpus, mode, kernel):
    c = b200_cluster(gpus)
    src = placement(gpus, *sp[:3], qkv=sp[3], gate_up=sp[4])
    dst = placement(gpus, *dp[:3], qkv=dp[3], gate_up=dp[4])
    plan = plan_param_realloc(model, src, dst, c, BALANCED if gpus == 8 else SPEC)
    sbufs = {d: Guarded(plan.shard_bytes(R.SRC, d)) for d in plan.devices(R.SRC)}
    dbufs = {d: Guarded(plan.shard_bytes(R.DST, d)) for d in plan.devices(R.DST)}
    try:
        for d, g in sbufs.items():
            R.fill_shard(plan, R.SRC, d, g.ptr, 17)
        ex = R.Executor(plan, 0, {d: g.ptr for d, g in sbufs.items()}, {d: g.ptr for d, g in dbufs.items()},
                        range(gpus), mode, chunk_bytes=1536)
        ex.set_kernel(kernel)
        ex.launch()
        R.stream_sync()
        for d, g in list(dbufs.items()) + list(sbufs.items()):
            before, body, after = g.read()
            assert (before == 0xA5A5).all() and (after == 0xA5A5).all(), f"guard of device {d} overwritten"
        for d, g in dbufs.items():
            assert np.array_equal(g.read()[1], O.fill(model, dst, c, d, 17)), d
        ex.close()
    finally:
        for g in list(sbufs.values()) + list(dbufs.values()):
            g.buf.free()
