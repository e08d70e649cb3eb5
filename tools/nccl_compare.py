#!/usr/bin/env python
"""NCCL comparison for the DP fan-out and stage-remap workloads.

The upstream runtime moves weights with NCCL broadcasts. The
NCCL baseline here does the standard thing: move whole source shards with a
collective — ``all_gather_into_tensor`` when every GPU holds sources (tp->dp),
``broadcast`` when one GPU holds the only replica — then unpack locally with
the library's pull executor (the K1 relayout) into the destination layout.
Times are CUDA events around collective + unpack, max over ranks; the result
is verified on device. Run with torchrun, one process per GPU:

  torchrun --nproc-per-node N tools/nccl_compare.py --workload llama7b_tp8_dp8_roundtrip
  torchrun --nproc-per-node N tools/nccl_compare.py --workload llama13b_pp2tp4_to_dp2tp4 --kind p2p
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2406_14088_b200 import runtime as R  # noqa: E402
from paper_2406_14088_b200.rlplan import BALANCED, plan_param_realloc  # noqa: E402
from paper_2406_14088_b200.workloads import WORKLOADS  # noqa: E402


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="llama7b_tp8_dp8_roundtrip")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--kind", choices=["auto", "p2p"], default="auto",
                    help="auto: broadcast (one source) or all_gather; p2p: send/recv of whole source shards")
    args = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = WORKLOADS[args.workload]
    c = w.cluster()
    src_p, dst_p = w.phases[0]
    plan = plan_param_realloc(w.model, src_p, dst_p, c, BALANCED)
    n = c.device_count()
    hosted = R.hosted_devices(n, rank, world)
    src_devs = plan.devices(R.SRC)
    sizes = {d: plan.shard_bytes(R.SRC, d) for d in src_devs}
    S = max(sizes.values())
    stream = torch.cuda.current_stream()
    if args.kind == "p2p":
        # Stage remap (e.g. 13B pp2 -> dp2): every source shard some remote
        # rank's destinations read is sent whole to that rank with NCCL
        # send/recv (exactly the needed bytes when TP is unchanged), then
        # unpacked locally by the pull executor.
        kind = "p2p"
        owner_of = {d: r for r in range(world) for d in R.hosted_devices(n, r, world)}
        need_from: dict = {}  # (src device, receiving rank) pairs
        for s_dev, dsts, _rects in plan.lowered():
            for d in dsts:
                if owner_of[d] != owner_of[s_dev]:
                    need_from[(s_dev, owner_of[d])] = True
        mine = {d: torch.zeros(sizes[d], dtype=torch.uint8, device="cuda") for d in src_devs if d in hosted}
        for d, t in mine.items():
            R.fill_shard(plan, R.SRC, d, t.data_ptr(), 7)
        recv = {s_dev: torch.zeros(sizes[s_dev], dtype=torch.uint8, device="cuda")
                for (s_dev, q) in need_from if q == rank}
        src_ptrs = {d: t.data_ptr() for d, t in mine.items()}
        src_ptrs.update({d: t.data_ptr() for d, t in recv.items()})
        sends = sorted((s_dev, q) for (s_dev, q) in need_from if owner_of[s_dev] == rank)
        recvs = sorted((s_dev, owner_of[s_dev]) for (s_dev, q) in need_from if q == rank)

        def collective():
            ops = [dist.P2POp(dist.isend, mine[s_dev], q) for (s_dev, q) in sends]
            ops += [dist.P2POp(dist.irecv, recv[s_dev], q) for (s_dev, q) in recvs]
            for w_ in dist.batch_isend_irecv(ops):
                w_.wait()
    elif len(src_devs) == 1:
        kind = "broadcast"
        d0 = src_devs[0]
        owner = d0 // (n // world)
        buf = torch.zeros(S, dtype=torch.uint8, device="cuda")
        if rank == owner:
            R.fill_shard(plan, R.SRC, d0, buf.data_ptr(), 7)
        src_ptrs = {d0: buf.data_ptr()}

        def collective():
            dist.broadcast(buf, src=owner)
    else:
        kind = "all_gather"
        mine = [d for d in src_devs if d in hosted]
        per_rank = len(mine)
        assert all(len([d for d in src_devs if d in R.hosted_devices(n, r, world)]) == per_rank
                   for r in range(world)), "uneven source hosting"
        assert len(set(sizes.values())) == 1, "all_gather needs equal shard sizes"
        local_in = torch.zeros(per_rank * S, dtype=torch.uint8, device="cuda")
        for i, d in enumerate(mine):
            R.fill_shard(plan, R.SRC, d, local_in.data_ptr() + i * S, 7)
        gathered = torch.zeros(world * per_rank * S, dtype=torch.uint8, device="cuda")
        order = [d for r in range(world) for d in src_devs if d in R.hosted_devices(n, r, world)]
        src_ptrs = {d: gathered.data_ptr() + i * S for i, d in enumerate(order)}

        def collective():
            dist.all_gather_into_tensor(gathered, local_in)
    dst = {d: R.DeviceBuffer(local, plan.shard_bytes(R.DST, d)) for d in plan.devices(R.DST) if d in hosted}
    for b in dst.values():
        b.zero()
    unpack = R.Executor(plan, local, src_ptrs, {d: b.ptr for d, b in dst.items()}, hosted, R.PULL)
    torch.cuda.synchronize()

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        collective()
        if ev:
            ev[1].record(stream)
        unpack.launch(stream)
        if ev:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    for k in range(args.steps):
        step(evs[k])
    torch.cuda.synchronize()
    coll = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    unp = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    total = sum(e[0].elapsed_time(e[2]) for e in evs) / args.steps
    bad = sum(R.verify_shard(plan, R.DST, d, b.ptr, 7)[0] for d, b in dst.items())
    t = torch.tensor([total, coll, unp, bad], dtype=torch.float64, device="cuda")
    mx = t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"impl": "nccl", "collective": kind, "workload": w.name, "n_gpus": world,
                          "ms": round(float(mx[0]), 4), "collective_ms": round(float(mx[1]), 4),
                          "unpack_ms": round(float(mx[2]), 4), "verified": float(mx[3]) == 0,
                          "nccl": ".".join(map(str, torch.cuda.nccl.version()))}), flush=True)
    unpack.close()
    for b in dst.values():
        b.free()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
