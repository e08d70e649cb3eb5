#!/usr/bin/env python
"""Concurrent pinned host->device bandwidth per GPU, with and without binding
each rank (and its pinned buffer) to the GPU's NUMA-local CPUs.

    torchrun --nproc-per-node N tools/h2d_numa.py [GiB per rank]

Prints one JSON line per mode from rank 0: per-rank GB/s when every rank
copies at once, plus the topology (NUMA node and CPU list of each GPU)."""
from __future__ import annotations

import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_14088_b200 import runtime as R  # noqa: E402


def gpu_numa(dev: int):
    p = torch.cuda.get_device_properties(dev)
    bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    base = f"/sys/bus/pci/devices/{bus}"
    try:
        node = int(open(f"{base}/numa_node").read())
        cpus = open(f"{base}/local_cpulist").read().strip()
    except OSError:
        node, cpus = None, None
    return bus, node, cpus


def parse_cpulist(s: str):
    out = set()
    for part in s.split(","):
        if "-" in part:
            a, b = part.split("-")
            out.update(range(int(a), int(b) + 1))
        elif part:
            out.add(int(part))
    return out


def measure(nbytes: int, dev: int, reps: int = 5, sync: bool = True):
    hb = R.HostBuffer(nbytes)
    db = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    R.memcpy_async(db.data_ptr(), hb.ptr, nbytes, 0, s)
    R.stream_sync(s)
    res = []
    for _ in range(reps):
        if sync:
            dist.barrier()
        t0 = time.perf_counter()
        R.memcpy_async(db.data_ptr(), hb.ptr, nbytes, 0, s)
        R.stream_sync(s)
        res.append(nbytes / (time.perf_counter() - t0) / 1e9)
    hb.free()
    del db
    return sorted(res)[len(res) // 2]


def main():
    gib = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    nbytes = int(gib * (1 << 30))
    bus, node, cpus = gpu_numa(dev)
    topo = [None] * world
    dist.all_gather_object(topo, {"rank": rank, "bus": bus, "numa": node, "cpus": cpus,
                                  "affinity_before": len(os.sched_getaffinity(0))})
    out = {}
    # unbound, all at once; then each rank alone; then bound to the GPU's node
    out["unbound_concurrent"] = measure(nbytes, dev)
    for r in range(world):
        dist.barrier()
        if r == rank:
            out["unbound_alone"] = measure(nbytes, dev, sync=False)
        dist.barrier()
    if cpus:
        os.sched_setaffinity(0, parse_cpulist(cpus))
    out["bound_concurrent"] = measure(nbytes, dev)
    for r in range(world):
        dist.barrier()
        if r == rank:
            out["bound_alone"] = measure(nbytes, dev, sync=False)
        dist.barrier()
    res = [None] * world
    dist.all_gather_object(res, out)
    if rank == 0:
        print(json.dumps({"world": world, "gib_per_rank": gib, "topo": topo,
                          "gbs": res,
                          "sum_unbound": round(sum(r["unbound_concurrent"] for r in res), 1),
                          "sum_bound": round(sum(r["bound_concurrent"] for r in res), 1)}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
