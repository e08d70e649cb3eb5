"""Fixed cost of one reallocation launch (1 GPU, BASELINE configs[0] tiny plan,
3.4 MB): host submission time of Executor.launch, GPU time of one launch
between events, and the per-launch time of 200 back-to-back launches.

    python tools/launch_latency.py  ->  one JSON line
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    import torch

    from paper_2406_14088_b200 import runtime as R
    from paper_2406_14088_b200.rlplan import BALANCED
    from paper_2406_14088_b200.workloads import WORKLOADS

    out = {}
    for name in ("tiny_tp2_to_dp2", "data_gen_dp8_to_pp2dp2tp2"):
        w = WORKLOADS[name]
        plan = w.plans(BALANCED)[0]
        vc = R.VirtualCluster(plan, 0)
        vc.fill_sources(1)
        stream = torch.cuda.current_stream()
        # chunk 0 = library default (small phases re-cut to ~one item per
        # resident CTA); 256 KiB = the fixed large-phase item size, for A/B
        for chunk, kernel in ((0, 0), (0, 1), (0, None), (256 << 10, None)):
            ex = vc.executor(R.PUSH, chunk, kernel)
            for _ in range(20):
                ex.launch(stream)
            torch.cuda.synchronize()
            # host submission cost per launch
            n = 200
            t0 = time.perf_counter()
            for _ in range(n):
                ex.launch(stream)
            host_us = (time.perf_counter() - t0) / n * 1e6
            torch.cuda.synchronize()
            # one launch between events, GPU idle before (what bench phase_ms sees)
            singles = []
            for _ in range(20):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                s.record(stream)
                ex.launch(stream)
                e.record(stream)
                torch.cuda.synchronize()
                singles.append(s.elapsed_time(e) * 1e3)
            # back to back, queued ahead: GPU time per launch
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(40_000_000)  # let the host queue everything first
            s.record(stream)
            for _ in range(n):
                ex.launch(stream)
            e.record(stream)
            torch.cuda.synchronize()
            out[f"{name}/kernel{'-default' if kernel is None else kernel}{'/chunk256k' if chunk else ''}"] = {"host_submit_us": round(host_us, 2),
                                            "single_event_us": round(sorted(singles)[len(singles) // 2], 2),
                                            "queued_gpu_us_per_launch": round(s.elapsed_time(e) * 1e3 / n, 2),
                                            "items": ex.items}
            ex.close()
        vc.free()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
