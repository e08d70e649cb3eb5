"""Pinned host -> device bandwidth per rank with one process per GPU
(diagnostics for the bench's e2e leg at N > 1).

Every rank allocates 4 GiB of pinned host memory, first-touches it, and
copies it to its GPU while the other ranks do the same. Run twice: as
launched (no CPU binding), and with each rank bound to its GPU's local CPUs
(/sys/bus/pci/devices/<bdf>/local_cpulist) before it allocates, so the
pinned pages land on the GPU's NUMA node.

    torchrun --nproc-per-node N tools/h2d_ranks.py
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def local_cpus(device: int):
    """CPUs on the NUMA node of GPU `device` (nvidia-smi bus id -> sysfs)."""
    import subprocess
    out = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", str(device)],
                         capture_output=True, text=True).stdout.strip().lower()
    dom, _, rest = out.partition(":")
    path = f"/sys/bus/pci/devices/{dom[-4:]}:{rest}/local_cpulist"
    try:
        text = open(path).read().strip()
    except OSError:
        return None, path
    cpus = set()
    for part in text.split(","):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    return cpus, path


def main() -> None:
    import torch
    import torch.distributed as dist

    from paper_2406_14088_b200 import runtime as R

    rank, world, lr = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(lr)
    dist.init_process_group("gloo")
    nbytes = 4 << 30
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    results = {}
    cpus, path = local_cpus(lr)
    stream = torch.cuda.current_stream()

    def timed_copy(h, n, turn=None):
        best = 1e30
        for _ in range(3):
            for r in range(world if turn else 1):
                dist.barrier()
                torch.cuda.synchronize()
                if turn and r != rank:
                    continue
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                R.memcpy_async(dev.data_ptr(), h.ptr, n, 0, stream)
                e.record(stream)
                torch.cuda.synchronize()
                best = min(best, s.elapsed_time(e))
        return round(n / (best * 1e-3) / 1e9, 2)

    import ctypes
    import mmap
    cudart = ctypes.CDLL("libcudart.so.12") if False else None

    class Registered:
        """malloc-style anonymous mapping (transparent huge pages when
        `huge`), page-locked with cudaHostRegister."""

        def __init__(self, n, huge):
            self.mm = mmap.mmap(-1, n, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
            if huge:
                self.mm.madvise(mmap.MADV_HUGEPAGE)
            self.buf = (ctypes.c_char * n).from_buffer(self.mm)
            self.ptr = ctypes.addressof(self.buf)
            ctypes.memset(self.ptr, 1, n)
            rc = torch.cuda.cudart().cudaHostRegister(self.ptr, n, 0)
            assert int(rc) == 0, rc

        def free(self):
            torch.cuda.cudart().cudaHostUnregister(self.ptr)
            del self.buf
            self.mm.close()

    n = 2 << 30
    h = R.HostBuffer(n)
    h.array()[:] = 1  # first touch
    results["together_mallochost"] = timed_copy(h, n)
    results["alone_mallochost"] = timed_copy(h, n, turn=True)
    h.free()
    for huge in (False, True):
        g = Registered(n, huge)
        results[f"together_register{'_thp' if huge else ''}"] = timed_copy(g, n)
        g.free()
    results["cpus_local"] = f"{min(cpus)}-{max(cpus)} ({len(cpus)})" if cpus else None
    allr = [None] * world
    dist.all_gather_object(allr, (rank, lr, results))
    if rank == 0:
        for r in sorted(allr):
            print(json.dumps({"rank": r[0], "gpu": r[1], **r[2]}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
