"""Pinned host -> device from ONE process driving every GPU at once, with a
separate cudaMallocHost buffer per GPU (compare tools/h2d_ranks.py, where
each GPU has its own process)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2406_14088_b200 import runtime as R
    g = torch.cuda.device_count()
    n = 2 << 30
    devs, hosts, streams = [], [], []
    for d in range(g):
        torch.cuda.set_device(d)
        devs.append(torch.empty(n, dtype=torch.uint8, device=f"cuda:{d}"))
        h = R.HostBuffer(n)
        h.array()[:] = 1
        hosts.append(h)
        streams.append(torch.cuda.Stream(device=d))
    best = 1e30
    import time
    for _ in range(3):
        for d in range(g):
            torch.cuda.synchronize(d)
        t0 = time.perf_counter()
        for d in range(g):
            with torch.cuda.device(d):
                R.memcpy_async(devs[d].data_ptr(), hosts[d].ptr, n, 0, streams[d])
        for d in range(g):
            torch.cuda.synchronize(d)
        best = min(best, time.perf_counter() - t0)
    print(f"single process, {g} GPUs, separate 2 GiB pinned buffers: {n / best / 1e9:.2f} GB/s per GPU "
          f"({g * n / best / 1e9:.1f} total)", flush=True)


if __name__ == "__main__":
    main()
