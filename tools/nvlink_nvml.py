#!/usr/bin/env python
"""NVLink traffic of a command from the hardware counters (NVML), per GPU.

Reads NVML_FI_DEV_NVLINK_THROUGHPUT_{DATA,RAW}_{TX,RX} (KiB, cumulative) on
every link of every visible GPU before and after running the command, and
prints the deltas: payload bytes (DATA) and wire bytes including protocol
(RAW). Copy engines have no per-kernel ncu counter, so this is how the
copy-engine transport's link bytes are measured.

    python tools/nvlink_nvml.py [--expect BYTES] -- <command...>
"""
from __future__ import annotations

import json
import subprocess
import sys
import time

import pynvml as N

FIELDS = {"data_tx": N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, "data_rx": N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX,
          "raw_tx": N.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX, "raw_rx": N.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX}


def sample(handles, links=18):
    out = []
    for h in handles:
        tot = {k: 0 for k in FIELDS}
        for k, fid in FIELDS.items():
            reqs = [(fid, l) for l in range(links)]
            try:
                vals = N.nvmlDeviceGetFieldValues(h, reqs)
            except N.NVMLError:
                continue
            for v in vals:
                if v.nvmlReturn == 0:
                    tot[k] += int(v.value.ullVal) * 1024
        out.append(tot)
    return out


def main() -> int:
    args = sys.argv[1:]
    expect = None
    if args[:1] == ["--expect"]:
        expect = float(args[1])
        args = args[2:]
    if args[:1] == ["--"]:
        args = args[1:]
    N.nvmlInit()
    handles = [N.nvmlDeviceGetHandleByIndex(i) for i in range(N.nvmlDeviceGetCount())]
    a = sample(handles)
    t0 = time.time()
    rc = subprocess.call(args)
    dt = time.time() - t0
    time.sleep(1.0)  # counters settle
    b = sample(handles)
    res = {"cmd": " ".join(args), "rc": rc, "wall_s": round(dt, 2), "gpus": []}
    for i, (x, y) in enumerate(zip(a, b)):
        d = {k: y[k] - x[k] for k in FIELDS}
        d["raw_over_data_tx"] = round(d["raw_tx"] / d["data_tx"], 4) if d["data_tx"] else None
        d["raw_over_data_rx"] = round(d["raw_rx"] / d["data_rx"], 4) if d["data_rx"] else None
        if expect:
            d["data_tx_over_expected"] = round(d["data_tx"] / expect, 4)
        res["gpus"].append({"gpu": i, **d})
    print(json.dumps(res), flush=True)
    return rc


if __name__ == "__main__":
    sys.exit(main())
