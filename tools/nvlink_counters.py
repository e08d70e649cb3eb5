#!/usr/bin/env python
"""NVLink byte counters for the cross-GPU copy kernel (ncu evidence).

ncu must not wrap multi-rank commands, so this drives two GPUs from ONE
process (peer access, no IPC): the 7B train->gen forward (8 plan devices,
4 per GPU, hierarchical push) runs as GPU 0's phase-0 kernel, then GPU 1's
(host-synchronised, no barrier and no cross-GPU waits), then the two in-host
fan-outs; every destination shard is verified. Under ncu, collect
nvltx/nvlrx user bytes per launch and compare with the library's wire
accounting printed here:

  python tools/nvlink_counters.py
  ncu --metrics nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,\
dram__bytes_write.sum,gpu__time_duration.sum -k regex:"rr_bulk_kernel|rr_copy_kernel" --csv \
python tools/nvlink_counters.py
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2406_14088_b200 import runtime as R  # noqa: E402
from paper_2406_14088_b200._lib import check, lib  # noqa: E402
from paper_2406_14088_b200.rlplan import BALANCED, plan_param_realloc  # noqa: E402
from paper_2406_14088_b200.workloads import WORKLOADS  # noqa: E402


def main() -> int:
    w = WORKLOADS["llama7b_tp8_dp8_roundtrip"]
    c = w.cluster()
    src_p, dst_p = w.phases[0]
    plan = plan_param_realloc(w.model, src_p, dst_p, c, BALANCED)
    gpus = 2
    host_of = [d // (8 // gpus) for d in range(8)]
    check(lib.rr_enable_peer(0, 1))
    check(lib.rr_enable_peer(1, 0))
    train = {d: R.DeviceBuffer(host_of[d], plan.shard_bytes(R.SRC, d)) for d in range(8)}
    gen = {d: R.DeviceBuffer(host_of[d], plan.shard_bytes(R.DST, d)) for d in range(8)}
    for d in range(8):
        R.fill_shard(plan, R.SRC, d, train[d].ptr, 9)
    execs = []
    for g in range(gpus):
        local = [d for d in range(8) if host_of[d] == g]
        ex = R.Executor(plan, g, {d: train[d].ptr for d in local}, {d: b.ptr for d, b in gen.items()}, local,
                        R.PUSH, host_of=host_of)
        execs.append(ex)
    import torch
    report = {}
    for rep in range(2):  # second round is the one to read in ncu (warm)
        for g, ex in enumerate(execs):
            torch.cuda.set_device(g)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            ex.launch()
            e.record()
            torch.cuda.synchronize(g)
            report[f"gpu{g}_phase0_ms"] = s.elapsed_time(e)
        for g, ex in enumerate(execs):
            torch.cuda.set_device(g)
            ex.launch_fanout()
            torch.cuda.synchronize(g)
    bad = sum(R.verify_shard(plan, R.DST, d, gen[d].ptr, 9)[0] for d in range(8))
    for g, ex in enumerate(execs):
        report[f"gpu{g}_wire_out_bytes"] = ex.wire_out
        report[f"gpu{g}_wire_in_bytes"] = ex.wire_in
        report[f"gpu{g}_phase0_hbm_bytes"] = ex.bytes_read + ex.bytes_written
    report["verified"] = bad == 0
    print(json.dumps(report), flush=True)
    for ex in execs:
        ex.close()
    for b in list(train.values()) + list(gen.values()):
        b.free()
    return 0 if bad == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
