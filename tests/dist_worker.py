"""Multi-process GPU parity worker (launched by tests/test_multigpu.py via
torchrun, one process per GPU). Each rank hosts a contiguous block of the 8
plan devices; destination shards of remote ranks are reached through CUDA
IPC and written by NVLink peer stores. Every rank compares its hosted
destination shards with the CPU oracle and the results are all-reduced."""
from __future__ import annotations

import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from _helpers import placement  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2406_14088_b200 import runtime as R  # noqa: E402
from paper_2406_14088_b200.rlplan import (BALANCED, MODELS, DeviceMesh, ParallelStrategy, Placement,  # noqa: E402
                                          b200_cluster, plan_param_realloc)
from paper_2406_14088_b200.workloads import WORKLOADS  # noqa: E402

TINY_GQA = dataclasses.replace(MODELS["tiny"], name="tiny_gqa", hidden_size=512, num_attention_heads=16,
                               num_kv_heads=8, intermediate_size=1024)

CASES = [
    ((1, 1, 8, 0, 0), (1, 8, 1, 0, 0)),
    ((4, 1, 2, 2, 1), (1, 1, 8, 1, 1)),
    ((2, 1, 4, 0, 0), (1, 1, 8, 0, 0)),
    ((2, 1, 4, 0, 0), (1, 2, 4, 0, 0)),
    ((1, 8, 1, 2, 1), (4, 1, 2, 0, 0)),
]


def main() -> int:
    rank, world, lrank = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    # More ranks than GPUs (e.g. world 8 on a 4-GPU box, the 8-GPU code path):
    # two processes share a GPU, their kernels time-slice, IPC and flags work
    # as across GPUs. NCCL refuses two ranks per GPU, so gloo carries the
    # host-side collectives; multicast needs distinct GPUs and is skipped.
    gpus = torch.cuda.device_count()
    local = lrank % gpus
    oversub = world > gpus
    torch.cuda.set_device(local)
    if oversub:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = b200_cluster(8)
    failures = []
    combos = [(m, k, h) for m in (R.PUSH, R.PULL) for k in (0, 1) for h in (True, False)]
    for mode, kernel, hier in combos:
        for sp, dp in CASES:
            src = placement(8, *sp[:3], qkv=sp[3], gate_up=sp[4])
            dst = placement(8, *dp[:3], qkv=dp[3], gate_up=dp[4])
            plan = plan_param_realloc(TINY_GQA, src, dst, c, BALANCED)
            rr = R.RankRealloc([plan], {"a": (0, R.SRC), "b": (0, R.DST)}, [("a", "b")], rank, world, local,
                               mode=mode, kernel=kernel, hierarchical=hier)
            for d, b in rr.buffers["a"].items():
                R.fill_shard(plan, R.SRC, d, b.ptr, 21)
            torch.cuda.synchronize()
            dist.barrier()
            rr.run_phase(0)
            torch.cuda.synchronize()
            if rr.barrier.timed_out():
                failures.append(f"{sp}->{dp} mode {mode} kernel {kernel} hier {hier}: barrier timed out")
            for d, b in rr.buffers["b"].items():
                got = b.to_host()
                want = O.fill(TINY_GQA, dst, c, d, 21)
                if not np.array_equal(got, want):
                    failures.append(f"{sp}->{dp} mode {mode} kernel {kernel} hier {hier}: device {d} differs in "
                                    f"{int(np.count_nonzero(got != want))} elements")
            dist.barrier()
            rr.close()
    # NVLS multicast (K3): one-to-many payloads stored once through multimem.st.
    if R.multicast_supported(local) and not oversub:
        mc_cases = [
            (Placement(DeviceMesh(0, 1, 0, 1), ParallelStrategy()), placement(8, 1, 8, 1)),  # replicate from dev 0
            (placement(8, 1, 1, 8), placement(8, 1, 8, 1)),                                  # tp8 -> dp8
        ]
        for src, dst in mc_cases:
            plan = plan_param_realloc(TINY_GQA, src, dst, c, BALANCED)
            rr = R.RankRealloc([plan], {"a": (0, R.SRC), "b": (0, R.DST)}, [("a", "b")], rank, world, local,
                               multicast=["b"])
            uses_mc = sum(e.stats(0)[0] for e in rr.executors) > 0
            for d, b in rr.buffers["a"].items():
                R.fill_shard(plan, R.SRC, d, b.ptr, 23)
            torch.cuda.synchronize()
            dist.barrier()
            rr.run_phase(0)
            torch.cuda.synchronize()
            for d, b in rr.buffers["b"].items():
                got = b.to_host()
                want = O.fill(TINY_GQA, dst, c, d, 23)
                if not np.array_equal(got, want):
                    failures.append(f"multicast {src.strategy}->{dst.strategy}: device {d} differs in "
                                    f"{int(np.count_nonzero(got != want))} elements (items {uses_mc})")
            rr.close()
    elif rank == 0:
        print("dist_worker: NVLS multicast not supported or GPUs shared, skipped", flush=True)
    # Overlapped fan-out (star flags) and relay + overlap, over all parity
    # cases, on the TMA bulk kernel (1) and the LDG/STG kernel (0).
    for relay_opt, kernel in ((False, 1), (True, 1), (False, 0), (True, 0)):
        for sp, dp in CASES:
            src = placement(8, *sp[:3], qkv=sp[3], gate_up=sp[4])
            dst = placement(8, *dp[:3], qkv=dp[3], gate_up=dp[4])
            plan = plan_param_realloc(TINY_GQA, src, dst, c, BALANCED)
            rr = R.RankRealloc([plan], {"a": (0, R.SRC), "b": (0, R.DST)}, [("a", "b")], rank, world, local,
                               relay=relay_opt, overlap=True, kernel=kernel, flag_kernel=kernel)
            for d, b in rr.buffers["a"].items():
                R.fill_shard(plan, R.SRC, d, b.ptr, 37)
            for rep in range(2):
                for b in rr.buffers["b"].values():
                    b.zero()
                torch.cuda.synchronize()
                dist.barrier()
                rr.run_phase(0)
                torch.cuda.synchronize()
                for d, b in rr.buffers["b"].items():
                    got = b.to_host()
                    want = O.fill(TINY_GQA, dst, c, d, 37)
                    if not np.array_equal(got, want):
                        failures.append(f"overlap relay={relay_opt} kernel {kernel} {sp}->{dp} rep {rep}: device {d} differs in "
                                        f"{int(np.count_nonzero(got != want))} elements")
            if rr.relay_timeouts():
                failures.append(f"overlap relay={relay_opt} kernel {kernel} {sp}->{dp}: {rr.relay_timeouts()} timeouts")
            rr.close()
    # Pipelined relay: chunks travel source -> GPU -> GPU with per-chunk flags.
    relay_cases = [
        (Placement(DeviceMesh(0, 1, 0, 1), ParallelStrategy()), placement(8, 1, 8, 1)),  # replicate from dev 0
        (placement(8, 1, 1, 8), placement(8, 1, 8, 1)),                                  # tp8 -> dp8
        (placement(2, 1, 1, 2, offset=2), placement(8, 1, 4, 2)),                        # 2 sources -> dp4 tp2
    ]
    for (src, dst), kernel in [(case, k) for case in relay_cases for k in (1, 0)]:
        plan = plan_param_realloc(TINY_GQA, src, dst, c, BALANCED)
        rr = R.RankRealloc([plan], {"a": (0, R.SRC), "b": (0, R.DST)}, [("a", "b")], rank, world, local,
                           relay=True, kernel=kernel, flag_kernel=kernel)
        for d, b in rr.buffers["a"].items():
            R.fill_shard(plan, R.SRC, d, b.ptr, 29)
        torch.cuda.synchronize()
        dist.barrier()
        for rep in range(3):  # epochs advance per launch
            for b in rr.buffers["b"].values():
                b.zero()
            torch.cuda.synchronize()
            dist.barrier()
            rr.run_phase(0)
            torch.cuda.synchronize()
            for d, b in rr.buffers["b"].items():
                got = b.to_host()
                want = O.fill(TINY_GQA, dst, c, d, 29)
                if not np.array_equal(got, want):
                    failures.append(f"relay kernel {kernel} {src.strategy}->{dst.strategy} rep {rep}: device {d} differs in "
                                    f"{int(np.count_nonzero(got != want))} elements")
        if rr.relay_timeouts():
            failures.append(f"relay kernel {kernel} {src.strategy}->{dst.strategy}: {rr.relay_timeouts()} timeouts")
        rr.close()
    # Fuzz: random placement pairs with random delivery options (same seed on
    # every rank, so all ranks build the same plans and executors).
    import random

    from _helpers import random_placement
    rng = random.Random(int(os.environ.get("RR_FUZZ_SEED", "2406")))
    fuzz_models = [TINY_GQA, dataclasses.replace(TINY_GQA, name="tiny_mqa", num_attention_heads=8, num_kv_heads=1,
                                                 num_layers=3)]
    ce_cases = 0  # fuzz cases in which this rank issued copy-engine runs
    staged_cases = 0  # fuzz cases with a staged-gather phase
    for i in range(int(os.environ.get("RR_FUZZ_CASES", "24"))):
        fm = fuzz_models[i % 2]
        src, dst = random_placement(rng, fm), random_placement(rng, fm)
        mode = rng.choice([R.PUSH, R.PULL])
        hier = rng.random() < 0.7
        relay = rng.choice([False, True, "auto"])
        overlap = rng.random() < 0.5
        kernel = rng.choice([0, 1, 5])
        chunk = rng.choice([0, 8192, 65536])
        ce = rng.choice([-1, 0, 4096])  # copy-engine runs: off, default (256 MiB: none here), >= 4 KiB
        staged = rng.random() < 0.25    # staged gather (push mode, hierarchical, no relay), 32 KiB pieces
        plan = plan_param_realloc(fm, src, dst, c, rng.choice([0, 1]))
        rr = R.RankRealloc([plan], {"a": (0, R.SRC), "b": (0, R.DST)}, [("a", "b")], rank, world, local,
                           mode=mode, kernel=kernel, flag_kernel=kernel, hierarchical=hier, relay=relay,
                           overlap=overlap, chunk_bytes=chunk, ce_min_run_bytes=ce, staged=staged,
                           stage_chunk_bytes=32 << 10)
        ce_cases += int(any(e.ce_runs()[0] for e in rr.executors))
        staged_cases += int(bool(rr.staged_phases))
        for d, b in rr.buffers["a"].items():
            R.fill_shard(plan, R.SRC, d, b.ptr, 50 + i)
        for rep in range(2):
            for b in rr.buffers["b"].values():
                b.zero()
            torch.cuda.synchronize()
            dist.barrier()
            rr.run_phase(0)
            torch.cuda.synchronize()
            for d, b in rr.buffers["b"].items():
                got = b.to_host()
                want = O.fill(fm, dst, c, d, 50 + i)
                if not np.array_equal(got, want):
                    failures.append(f"fuzz {i} {src}->{dst} mode {mode} hier {hier} relay {relay} overlap {overlap} "
                                    f"kernel {kernel} chunk {chunk} ce {ce} staged {rr.staged_phases} rep {rep}: device {d} differs in "
                                    f"{int(np.count_nonzero(got != want))} elements")
        if rr.relay_timeouts() or rr.barrier.timed_out():
            failures.append(f"fuzz {i}: flag or barrier timeouts")
        dist.barrier()
        rr.close()
    # Copy-engine runs on stage remaps (forced down to 4 KiB ranges so the
    # tiny model has some), push and hierarchical/flat, with the onload path.
    ce_total = 0
    for sp, dp in (((2, 1, 4, 0, 0), (1, 2, 4, 0, 0)), ((2, 2, 2, 1, 1), (1, 4, 2, 1, 1)),
                   ((1, 2, 4, 2, 1), (2, 1, 4, 2, 1))):
        for hier in (True, False):
            src = placement(8, *sp[:3], qkv=sp[3], gate_up=sp[4])
            dst = placement(8, *dp[:3], qkv=dp[3], gate_up=dp[4])
            plan = plan_param_realloc(TINY_GQA, src, dst, c, BALANCED)
            rr = R.RankRealloc([plan], {"a": (0, R.SRC), "b": (0, R.DST)}, [("a", "b")], rank, world, local,
                               hierarchical=hier, ce_min_run_bytes=4096)
            ce_total += sum(e.ce_runs()[0] for e in rr.executors)
            for d, b in rr.buffers["a"].items():
                R.fill_shard(plan, R.SRC, d, b.ptr, 77)
            for onload in (False, True):
                for b in rr.buffers["b"].values():
                    b.zero()
                torch.cuda.synchronize()
                dist.barrier()
                if onload:
                    host = {d: R.HostBuffer(plan.shard_bytes(R.SRC, d)) for d in rr.buffers["a"]}
                    for d, hb in host.items():
                        hb.array()[:] = rr.buffers["a"][d].to_host()
                    copy_stream = torch.cuda.Stream()
                    # small chunks so that runs straddle several of them
                    rr.run_phase_onload(0, {d: hb.ptr for d, hb in host.items()}, copy_stream, chunk_bytes=64 << 10)
                else:
                    rr.run_phase(0)
                torch.cuda.synchronize()
                for d, b in rr.buffers["b"].items():
                    bad, first = R.verify_shard(plan, R.DST, d, b.ptr, 77)
                    if bad:
                        failures.append(f"ce {sp}->{dp} hier {hier} onload {onload}: device {d} {bad} mismatches")
                if onload:
                    for hb in host.values():
                        hb.free()
            if rr.barrier.timed_out():
                failures.append(f"ce {sp}->{dp}: barrier timed out")
            dist.barrier()
            rr.close()
    # Staged gather (copy-engine rotation + per-piece unpack), small pieces.
    staged_total = 0
    for sp, dp in (((1, 1, 8, 0, 0), (1, 8, 1, 0, 0)), ((2, 1, 4, 1, 1), (1, 1, 8, 0, 0)),
                   ((1, 2, 4, 0, 0), (4, 1, 2, 2, 1)), ((1, 8, 1, 0, 0), (1, 1, 8, 0, 0))):
        src = placement(8, *sp[:3], qkv=sp[3], gate_up=sp[4])
        dst = placement(8, *dp[:3], qkv=dp[3], gate_up=dp[4])
        plan = plan_param_realloc(TINY_GQA, src, dst, c, BALANCED)
        rr = R.RankRealloc([plan], {"a": (0, R.SRC), "b": (0, R.DST)}, [("a", "b")], rank, world, local,
                           staged=True, stage_chunk_bytes=64 << 10)
        staged_total += len(rr.staged_phases)
        for d, b in rr.buffers["a"].items():
            R.fill_shard(plan, R.SRC, d, b.ptr, 91)
        for onload in (False, True, False):  # repeated launches exercise the flag epochs
            for b in rr.buffers["b"].values():
                b.zero()
            torch.cuda.synchronize()
            dist.barrier()
            if onload:
                host = {d: R.HostBuffer(plan.shard_bytes(R.SRC, d)) for d in rr.buffers["a"]}
                for d, hb in host.items():
                    hb.array()[:] = rr.buffers["a"][d].to_host()
                rr.run_phase_onload(0, {d: hb.ptr for d, hb in host.items()}, torch.cuda.Stream(),
                                    chunk_bytes=64 << 10)
            else:
                rr.run_phase(0)
            torch.cuda.synchronize()
            for d, b in rr.buffers["b"].items():
                bad, first = R.verify_shard(plan, R.DST, d, b.ptr, 91)
                if bad:
                    failures.append(f"staged {sp}->{dp} onload {onload}: device {d} {bad} mismatches")
            if onload:
                for hb in host.values():
                    hb.free()
        if rr.relay_timeouts() or rr.barrier.timed_out():
            failures.append(f"staged {sp}->{dp}: flag or barrier timeouts")
        dist.barrier()
        rr.close()
    if world > 1 and staged_total == 0:
        failures.append("staged cases ran no staged phase")
    if world > 1 and not oversub:
        t = torch.tensor([ce_total], device="cuda")
        dist.all_reduce(t)
        if t.item() == 0:
            failures.append("copy-engine cases issued no runs")
    if os.environ.get("RR_FULL_7B") == "1" and not oversub:
        w = WORKLOADS["llama7b_tp8_dp8_roundtrip"]
        plans = [plan_param_realloc(w.model, s, d, c, BALANCED) for (s, d) in w.phases]
        rr = R.RankRealloc(plans, {"train": (0, R.SRC), "gen": (0, R.DST)}, [("train", "gen"), ("gen", "train")],
                           rank, world, local)
        for d, b in rr.buffers["train"].items():
            R.fill_shard(plans[0], R.SRC, d, b.ptr, 4)
        torch.cuda.synchronize()
        dist.barrier()
        for _ in range(2):
            rr.run_phase(0)
            rr.run_phase(1)
        torch.cuda.synchronize()
        for name, p in (("gen", plans[0]), ("train", plans[1])):
            for d, b in rr.buffers[name].items():
                bad, first = R.verify_shard(p, R.DST, d, b.ptr, 4)
                if bad:
                    failures.append(f"7B {name} shard {d}: {bad} mismatches (first {first})")
        dist.barrier()
        rr.close()
    flag = torch.tensor([len(failures)], device="cpu" if oversub else "cuda")
    dist.all_reduce(flag)
    for f in failures:
        print(f"rank {rank}: {f}", flush=True)
    if rank == 0:
        print(f"dist_worker: fuzz cases with copy-engine runs on rank 0: {ce_cases}, staged: {staged_cases}",
              flush=True)
        print(f"dist_worker world={world}: {'OK' if flag.item() == 0 else 'FAILED'}", flush=True)
    dist.destroy_process_group()
    return 0 if flag.item() == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
