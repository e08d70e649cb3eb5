#!/usr/bin/env python
"""One process per GPU: reshard an actor's weights from its training layout
to its generation layout and back, the way a ReaL-style runtime would call
the library between a training and a generation call.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 examples/rank_realloc.py [--model llama7b]

Every rank hosts (plan devices / world) plan devices. The training shards are
filled with the library's hash weights, the phases run (the delivery scheme
of each is picked by timing the candidates on these buffers), and every
destination shard is checked on the device against the expected values.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_14088_b200 import runtime as R  # noqa: E402
from paper_2406_14088_b200.rlplan import (BALANCED, MODELS, DeviceMesh, ParallelStrategy,  # noqa: E402
                                          Placement, b200_cluster, plan_param_realloc)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama7b", choices=sorted(MODELS))
    ap.add_argument("--devices", type=int, default=8, help="plan devices (spread over the ranks)")
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    gpu = int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    if world > 1:
        # gloo when ranks share a GPU (NCCL refuses that), else NCCL
        shared = world > torch.cuda.device_count()
        dist.init_process_group("gloo" if shared else "nccl",
                                **({} if shared else {"device_id": torch.device("cuda", gpu)}))

    n = args.devices
    cluster = b200_cluster(n)
    mesh = DeviceMesh(0, 1, 0, n)
    train = Placement(mesh, ParallelStrategy(tp=n))
    gen = Placement(mesh, ParallelStrategy(dp=n))
    model = MODELS[args.model]
    plans = [plan_param_realloc(model, train, gen, cluster, BALANCED),
             plan_param_realloc(model, gen, train, cluster, BALANCED)]

    # shard sets: phase 0 reads "train" and writes "gen"; phase 1 writes "train" back
    rr = R.RankRealloc(plans, {"train": (0, R.SRC), "gen": (0, R.DST)}, [("train", "gen"), ("gen", "train")],
                       rank, world, gpu, relay="auto", overlap=True, staged="auto",
                       ce_transport="auto", probe=world > 1)
    seed = 7
    for d, b in rr.buffers["train"].items():
        R.fill_shard(plans[0], R.SRC, d, b.ptr, seed)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    t = []
    for _ in range(args.steps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(len(plans)):
            rr.run_phase(i, stream)
        torch.cuda.synchronize()
        t.append((time.perf_counter() - t0) * 1e3)

    bad = 0
    for d, b in rr.buffers["gen"].items():
        bad += R.verify_shard(plans[0], R.DST, d, b.ptr, seed)[0]
    for d, b in rr.buffers["train"].items():
        bad += R.verify_shard(plans[1], R.DST, d, b.ptr, seed)[0]
    nccl = world > 1 and dist.get_backend() == "nccl"
    tot = torch.tensor([bad], dtype=torch.int64, device="cuda" if nccl else "cpu")
    if world > 1:
        dist.all_reduce(tot)
    schemes = [s.label() for s in rr.schemes]
    rr.close()
    if rank == 0:
        print(f"{args.model} tp{n} -> dp{n} -> tp{n} on {world} rank(s): {min(t):.2f} ms per round trip "
              f"(best of {args.steps}), schemes {schemes}, mismatches {int(tot.item())}", flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0 if int(tot.item()) == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
