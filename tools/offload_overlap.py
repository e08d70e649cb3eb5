"""Offload overlapped with the reallocation, 1 GPU.

LLaMA-7B train (pp1,dp1,tp8) -> gen (pp1,dp8,tp1) over 8 plan devices. Times
(a) the reallocation alone, (b) parking the 16.06 GB of training shards in
pinned host memory alone, (c) both through RankRealloc.run_phase_offload,
where the device->host copies and the copy kernels read the same shards.
Checks the parked bytes and the generation shards afterwards.

    python tools/offload_overlap.py  ->  one JSON line
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    import numpy as np
    import torch

    from paper_2406_14088_b200 import runtime as R
    from paper_2406_14088_b200.rlplan import BALANCED
    from paper_2406_14088_b200.workloads import WORKLOADS

    w = WORKLOADS["llama7b_tp8_dp8_roundtrip"]
    plan = w.plans(BALANCED)[0]
    rr = R.RankRealloc([plan], {"train": (0, R.SRC), "gen": (0, R.DST)}, [("train", "gen")], 0, 1, 0)
    stream = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    for d, b in rr.buffers["train"].items():
        R.fill_shard(plan, R.SRC, d, b.ptr, 3)
    host = {d: R.HostBuffer(b.nbytes) for d, b in rr.buffers["train"].items()}
    hp = {d: h.ptr for d, h in host.items()}
    src_bytes = {d: b.nbytes for d, b in rr.buffers["train"].items()}

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            fn()
            done = torch.cuda.Event()
            done.record(copy)
            stream.wait_event(done)  # the step ends when both streams are done
            e.record(stream)
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e))
        return best

    realloc = timed(lambda: rr.run_phase(0, stream))
    offload = timed(lambda: rr.executors[0].launch_offload(src_bytes, hp, copy, stream))
    both = timed(lambda: rr.run_phase_offload(0, hp, copy, stream))
    bad = sum(R.verify_shard(plan, R.DST, d, b.ptr, 3)[0] for d, b in rr.buffers["gen"].items())
    # parked bytes: compare against the shards still on the device
    ok_host = True
    for d, b in rr.buffers["train"].items():
        dev = np.empty(b.nbytes // 2, np.uint16)
        R.check(R.lib.rr_memcpy(dev.ctypes.data, b.ptr, b.nbytes, 1, None, 1))
        ok_host = ok_host and np.array_equal(dev, host[d].array())
    gb = sum(src_bytes.values()) / 1e9
    print(json.dumps({"workload": w.name + " forward", "realloc_ms": round(realloc, 3),
                      "offload_ms": round(offload, 3), "offload_gbs": round(gb / (offload * 1e-3), 2),
                      "overlapped_ms": round(both, 3), "hidden_fraction_of_realloc":
                          round(1 - (both - offload) / realloc, 3),
                      "parked_bytes": int(sum(src_bytes.values())), "parked_ok": ok_host,
                      "gen_shards_ok": bad == 0}), flush=True)
    for h in host.values():
        h.free()
    rr.close()


if __name__ == "__main__":
    main()
