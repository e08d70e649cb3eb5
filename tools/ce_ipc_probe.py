"""Copy engine over CUDA IPC, one process per GPU (diagnostics). Each rank
copies into its partner's (rank ^ 1) IPC-mapped buffer with cudaMemcpyAsync
while the partner does the same; GB/s per GPU per direction, max over ranks.

    torchrun --nproc-per-node 2 tools/ce_ipc_probe.py
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2406_14088_b200 import runtime as R  # noqa: E402


def main() -> None:
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    G = 1 << 30
    big = int(os.environ.get("CE_PROBE_GIB", "8"))
    src = R.DeviceBuffer(local, big * G)
    dst = R.DeviceBuffer(local, big * G)
    src.zero()
    # CE_PROBE_RANDOM=1: random source bytes (the product's hash-initialised
    # weights) instead of zeros
    rnd = os.environ.get("CE_PROBE_RANDOM") == "1"
    if rnd:
        t = torch.empty(big * G // 8, dtype=torch.int64, device="cuda").random_()
        R.memcpy_async(src.ptr, t.data_ptr(), big * G, 2, None)
        torch.cuda.synchronize()
        del t
    handles = [None] * world
    dist.all_gather_object(handles, dst.ipc_handle())
    peer = rank ^ 1
    remote = R.open_ipc(local, handles[peer])
    stream = torch.cuda.Stream()
    out = {}

    def timed(name, fn, nbytes):
        best = 1e30
        for r in range(4):
            torch.cuda.synchronize()
            dist.barrier()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            fn()
            e.record(stream)
            torch.cuda.synchronize()
            if r:
                best = min(best, s.elapsed_time(e))
        t = torch.tensor([best], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[name] = round(nbytes / (t.item() * 1e6), 1)

    for size_gib in (1, 2, 3):
        n = size_gib * G
        timed(f"one_copy_{size_gib}GiB", lambda: R.memcpy_async(remote, src.ptr, n, 2, stream), n)
    timed("4x512MiB", lambda: [R.memcpy_async(remote + k * (G // 2), src.ptr + k * (G // 2), G // 2, 2, stream)
                               for k in range(4)], 2 * G)
    # misaligned runs, as the plan's ranges are (256-byte aligned offsets)
    for so, do in ((256, 256), (256, 0), (4096, 0), (65536, 0), (1 << 20, 0), (3 << 20, 1 << 20), (768, 4352)):
        n = 2 * G
        timed(f"2GiB_src+{so}_dst+{do}", lambda: R.memcpy_async(remote + do, src.ptr + so, n, 2, stream), n)
    # long copies across a large address range (the 13B stage remap moves 4 x 3.5 GB per GPU)
    run = 3500 * (1 << 20)
    if big >= 15:
        timed("1x3.5GB", lambda: R.memcpy_async(remote, src.ptr, run, 2, stream), run)
        timed("4x3.5GB_sequential", lambda: [R.memcpy_async(remote + k * run, src.ptr + k * run, run, 2, stream)
                                             for k in range(4)], 4 * run)
        timed("14GB_one_copy", lambda: R.memcpy_async(remote, src.ptr, 4 * run, 2, stream), 4 * run)
    # the 13B stage remap's pattern: 4 separate source buffers, 4 separate
    # (IPC-mapped) destination buffers, one 3.5 GB run each, runs at an offset
    srcs = [R.DeviceBuffer(local, run + (1 << 20)) for _ in range(4)]
    for b in srcs:
        R.memcpy_async(b.ptr, src.ptr, run, 2, None)
    dsts = [R.DeviceBuffer(local, 2 * run + (64 << 20)) for _ in range(4)]
    hs = [None] * world
    dist.all_gather_object(hs, [b.ipc_handle() for b in dsts])
    rem = [R.open_ipc(local, h) for h in hs[peer]]
    off = run + (13 << 20) + 256
    timed("4_buffers_4x3.5GB", lambda: [R.memcpy_async(rem[k] + off, srcs[k].ptr, run, 2, stream)
                                        for k in range(4)], 4 * run)
    timed("4_buffers_4x3.5GB_at0", lambda: [R.memcpy_async(rem[k], srcs[k].ptr, run, 2, stream)
                                            for k in range(4)], 4 * run)
    for p_ in rem:
        R.close_ipc(p_)
    for b in srcs + dsts:
        b.free()
    timed("local_d2d_2GiB", lambda: R.memcpy_async(dst.ptr, src.ptr, 2 * G, 2, stream), 4 * G)
    if rank == 0:
        print(json.dumps({"world": world, "random_source": rnd, "GBps_per_gpu_per_direction": out}), flush=True)
    dist.barrier()
    R.close_ipc(remote)
    src.free()
    dst.free()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
