#!/usr/bin/env python
"""NVLink ceilings on 2 GPUs: copy engine (CE) peer copies vs the SM push.

Measures what the copy engines reach over NVLink 5 for the transfer shapes
the reallocation produces, to decide whether big contiguous cross-GPU runs
should go to the CEs (cudaMemcpyAsync / cudaMemcpy2DAsync on side streams)
instead of SM peer stores:
  ce_uni     one 1D copy GPU0 -> GPU1
  ce_bi      GPU0 -> GPU1 and GPU1 -> GPU0 at once (the all-gather case)
  ce_bi_s4   the same split over 4 streams per GPU
  ce_bi_64M  the same as 64 MiB copies (per-copy overhead)
  ce2d_bi    strided destination rows (1 KiB of every 8 KiB, the row-parallel
             `o` shard landing in a dp replica)
  ce_bi+hbm  ce_bi while each GPU also runs a local HBM copy (the in-host
             fan-out running beside the NVLink transfer)
Every number is bytes crossing NVLink per GPU per direction / time, device
timed with CUDA events per GPU, max over the two GPUs.

  python tools/nvlink_ceiling.py  (needs 2 GPUs)
"""
from __future__ import annotations

import ctypes
import glob
import json
import os

import torch

GiB = 1 << 30


def cudart():
    import nvidia.cuda_runtime as m
    path = glob.glob(os.path.join(os.path.dirname(m.__file__), "lib", "libcudart.so*"))[0]
    rt = ctypes.CDLL(path)
    rt.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                     ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    return rt


def timed(work, devs, reps=5):
    """work(dev, stream) enqueues one repetition on `stream` of device dev."""
    streams = {d: torch.cuda.Stream(device=d) for d in devs}
    for d in devs:
        with torch.cuda.device(d):
            work(d, streams[d])
    best = None
    for _ in range(reps):
        for d in devs:
            torch.cuda.synchronize(d)
        ev = {}
        for d in devs:
            with torch.cuda.device(d):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(streams[d])
                work(d, streams[d])
                e.record(streams[d])
                ev[d] = (s, e)
        for d in devs:
            torch.cuda.synchronize(d)
        ms = max(s.elapsed_time(e) for s, e in ev.values())
        best = ms if best is None else min(best, ms)
    return best


def main() -> int:
    assert torch.cuda.device_count() >= 2, "needs 2 GPUs"
    rt = cudart()
    for a, b in ((0, 1), (1, 0)):
        with torch.cuda.device(a):
            if torch.cuda.can_device_access_peer(a, b):
                try:
                    torch.empty(1, device=f"cuda:{a}").to(f"cuda:{b}")
                except RuntimeError:
                    pass
    n = 4 * GiB
    src = {d: torch.empty(n, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)}
    dst = {d: torch.empty(n, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)}
    loc_a = {d: torch.empty(4 * GiB, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)}
    loc_b = {d: torch.empty(4 * GiB, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)}
    peer = {0: 1, 1: 0}
    out = {}

    def ce(d, s, nbytes=n, chunk=n):
        with torch.cuda.stream(s):
            for off in range(0, nbytes, chunk):
                m = min(chunk, nbytes - off)
                dst[peer[d]][off:off + m].copy_(src[d][off:off + m], non_blocking=True)

    ms = timed(lambda d, s: ce(d, s) if d == 0 else None, [0, 1])
    out["ce_uni_gbs"] = n / ms / 1e6
    ms = timed(ce, [0, 1])
    out["ce_bi_gbs"] = n / ms / 1e6
    ms = timed(lambda d, s: ce(d, s, chunk=64 << 20), [0, 1])
    out["ce_bi_64M_gbs"] = n / ms / 1e6

    side = {d: [torch.cuda.Stream(device=d) for _ in range(4)] for d in (0, 1)}

    def ce4(d, s):
        q = n // 4
        ev = torch.cuda.Event()
        ev.record(s)
        for i, t in enumerate(side[d]):
            t.wait_event(ev)
            with torch.cuda.stream(t):
                dst[peer[d]][i * q:(i + 1) * q].copy_(src[d][i * q:(i + 1) * q], non_blocking=True)
            e2 = torch.cuda.Event()
            e2.record(t)
            s.wait_event(e2)

    ms = timed(ce4, [0, 1])
    out["ce_bi_s4_gbs"] = n / ms / 1e6

    width, pitch = 1024, 8192
    rows = n // pitch

    def ce2d(d, s):
        r = rt.cudaMemcpy2DAsync(ctypes.c_void_p(dst[peer[d]].data_ptr()), pitch, ctypes.c_void_p(src[d].data_ptr()),
                                 width, width, rows, 3, ctypes.c_void_p(s.cuda_stream))
        assert r == 0, r

    ms = timed(ce2d, [0, 1])
    out["ce2d_bi_gbs"] = width * rows / ms / 1e6
    out["ce2d_shape"] = f"{rows} rows x {width} B, dst pitch {pitch} B"

    def hbm(d, s):
        with torch.cuda.stream(s):
            loc_b[d].copy_(loc_a[d], non_blocking=True)

    ms = timed(hbm, [0, 1])
    out["hbm_copy_alone_gbs_rw"] = 2 * 4 * GiB / ms / 1e6

    # CE push and an SM-driven HBM copy side by side (different streams).
    other = {d: torch.cuda.Stream(device=d) for d in (0, 1)}

    def both(d, s):
        ev = torch.cuda.Event()
        ev.record(s)
        other[d].wait_event(ev)
        with torch.cuda.stream(other[d]):
            loc_b[d].copy_(loc_a[d], non_blocking=True)
        ce(d, s)
        e2 = torch.cuda.Event()
        e2.record(other[d])
        s.wait_event(e2)

    ms = timed(both, [0, 1])
    out["ce_bi+hbm_ms"] = ms
    out["ce_bi+hbm_note"] = f"4 GiB over NVLink each way + 4 GiB local copy per GPU in {ms:.2f} ms"
    print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in out.items()}), flush=True)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
