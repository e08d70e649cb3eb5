#!/usr/bin/env python
"""Benchmark of the B200 parameter-reallocation path (ReaL, arXiv 2406.14088).

Metric (BASELINE.json): param realloc ms and per-GPU NVLink GB/s vs the
900 GB/s roofline. A step = one pass of the workload's phases; the default
workload is BASELINE.json configs[1] — LLaMA-7B bf16 train layout
(pp1,dp1,tp8) -> generation layout (pp1,dp8,tp1) and back — over 8 plan
devices hosted on N GPUs (8/N per GPU; at N=1 every move is a local HBM
relayout, at N=8 every remote slice crosses NVLink).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

`value` = bytes delivered into destination shards per second over the
whole job (all phases, all ranks), inputs resident in HBM; `ms_per_step`
is the realloc time of one step (max over ranks). `e2e` runs the same step
through the public API with the source shards onloaded from pinned host
memory inside the timed region. `--impl reference` times the reference's
CPU reallocation (the oracle restatement, oracle/, all host threads) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "param realloc ms and per-GPU NVLink GB/s (LLaMA-7B/70B) vs 900 GB/s roofline"
NVLINK_PEAK = 900.0  # GB/s per direction per GPU (nominal)


def measured_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(r[1]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# workloads as plain data, and the reference / CPU arm
# ---------------------------------------------------------------------------

def plain_workload(name: str):
    """A named workload of paper_2406_14088_b200/workloads.json as duck-typed
    objects with the reference types' attribute names (ModelSpec, Placement,
    DeviceMesh, ParallelStrategy, ClusterSpec), which the oracle accepts. The
    reference arm runs on these and never imports the product package."""
    from types import SimpleNamespace as NS
    with open(os.path.join(ROOT, "paper_2406_14088_b200", "workloads.json")) as f:
        table = json.load(f)
    e = next((w for w in table["workloads"] if w["name"] == name), None)
    if e is None:
        raise SystemExit(f"unknown workload {name!r}")
    model = NS(name=e["model"], **table["models"][e["model"]])

    def placement(d):
        no, nc, go, gc = d["mesh"]
        return NS(mesh=NS(node_offset=no, node_count=nc, gpu_offset=go, gpu_count=gc),
                  strategy=NS(dp=d["dp"], tp=d["tp"], pp=d["pp"]), qkv_layout=d.get("qkv_layout", 0),
                  gate_up_layout=d.get("gate_up_layout", 0), kv_layout=d.get("kv_layout", 0))
    src, dst = placement(e["src"]), placement(e["dst"])
    return NS(name=name, description=e["description"], model=model, devices=e["devices"],
              phases=[(src, dst), (dst, src)] if e["back"] else [(src, dst)], data_bytes=e.get("data_bytes", 0),
              cluster=NS(n_nodes=1, gpus_per_node=e["devices"], intra_node_bw=900e9, inter_node_bw=50e9))


L2_BYTES = 126 << 20  # B200 L2


def workload_config(w) -> dict:
    """`config` of the JSON line: the workload only (identical in both arms);
    how each arm executes it goes under `executor`."""
    def s(p):
        st = p.strategy
        return f"(pp{st.pp},dp{st.dp},tp{st.tp})"
    m = w.model
    h, hd = m.hidden_size, m.hidden_size // m.num_attention_heads
    params = (m.vocab_size * h * (2 if m.has_output_head else 1) + h +
              m.num_layers * (2 * h * h + 2 * h * hd * m.num_kv_heads + 3 * h * m.intermediate_size + 2 * h))
    nbytes = w.data_bytes * w.devices if w.data_bytes else params * m.param_bytes
    if nbytes > 2 * L2_BYTES:
        l2 = f"inputs larger than L2 ({nbytes / 1e9:.2f} GB of source shards per step); no flush needed"
    elif nbytes > L2_BYTES:
        l2 = f"{nbytes / 1e6:.1f} MB of source shards per step, under twice the 126 MB L2: partly L2-resident"
    else:
        l2 = (f"{nbytes / 1e6:.1f} MB of source shards: L2-resident across steps (a latency-bound parity "
              f"case, not a bandwidth measurement)")
    return {"workload": w.name, "description": w.description, "plan_devices": w.devices,
            "phases": [f"{s(a)}->{s(b)}" for a, b in w.phases],
            "l2": l2,
            "weights": "hash-initialised bf16 (seed 1); every destination shard checked after timing"}


def host_info() -> dict:
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), model)
    except OSError:
        pass
    return {"cpu_model": model, "cores": os.cpu_count() or 1, "mem_available_gb": round(mem_available() / 1e9, 1)}


def mem_available() -> int:
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except OSError:
        pass
    return 0


def cpu_realloc(w, steps: int, warmup: int, threads: int, budget_s: float = None) -> dict:
    """The reference path on the host: the oracle's CPU reallocation
    (oracle/liboracle.so, SPEC.md:541-611 restated; the reference itself
    moves no bytes) of the WHOLE workload `w` (plain objects),
    every phase per step, all shards in host RAM, `threads` worker threads.
    Steps run until both `steps` and (if given) `budget_s` are reached. The
    result is checked against the oracle's expected shards afterwards: the
    last phase's destinations byte for byte, earlier ones on 64 MiB windows."""
    import numpy as np
    from oracle import oracle as O
    c = w.cluster
    n = c.n_nodes * c.gpus_per_node
    if w.data_bytes:
        return cpu_data(w, steps, warmup, threads, budget_s)
    phases = []
    bufs = {}
    for (src, dst) in w.phases:
        ops, loc, _tb, _et = O.plan(w.model, src, dst, c, 1)  # 1 = balanced sources, as the B200 arm
        phases.append((src, dst, ops + loc))

    def key(p):
        return (p.strategy.pp, p.strategy.dp, p.strategy.tp, p.qkv_layout, p.gate_up_layout, p.kv_layout,
                p.mesh.gpu_offset, p.mesh.gpu_count)
    sets = {}
    for src, dst, _ops in phases:
        for p in (src, dst):
            sets.setdefault(key(p), p)
    need = sum(O.shard_bytes(w.model, p, c, d) for p in sets.values() for d in range(n))
    if need > 0.85 * mem_available():
        raise MemoryError(f"{w.name}: {need / 1e9:.1f} GB of shards, {mem_available() / 1e9:.1f} GB available")
    for k, p in sets.items():  # calloc'd: padding stays zero, pages fault in during warm-up
        bufs[k] = [np.zeros(O.shard_bytes(w.model, p, c, d) // 2, np.uint16) for d in range(n)]
    first = phases[0][0]
    for d in range(n):
        if bufs[key(first)][d].size:
            O.fill_range_into(w.model, first, c, d, 1, 0, bufs[key(first)][d].nbytes,
                              bufs[key(first)][d].ctypes.data, threads)
    delivered = sum(b * len(dsts) for (_s, _d, ops) in phases for (_src, dsts, _p, b) in ops)

    def step():
        for (src, dst, ops) in phases:
            O.execute(w.model, src, dst, c, ops, bufs[key(src)], bufs[key(dst)], threads)

    for _ in range(warmup):
        step()
    t0 = time.perf_counter()
    done = 0
    while True:
        step()
        done += 1
        el = time.perf_counter() - t0
        if done >= steps and (budget_s is None or el >= budget_s or done >= 100):
            break
    dt = (time.perf_counter() - t0) / done
    bad = 0
    for i, (_src, dst, _ops) in enumerate(phases):
        for d, b in enumerate(bufs[key(dst)]):
            if not b.size:
                continue
            n_check = b.nbytes if i == len(phases) - 1 else min(b.nbytes, 64 << 20)
            bad += O.check_range(w.model, dst, c, d, 1, 0, n_check, b.ctypes.data, threads)[0]
    return {"gbs": delivered / dt / 1e9, "s_per_step": dt, "delivered": delivered, "correct": bad == 0,
            "steps": done, "shard_gb": need / 1e9}


def cpu_data(w, steps: int, warmup: int, threads: int, budget_s: float = None) -> dict:
    """cpu_realloc for a data workload: the oracle's plan_data_transfer
    restatement executed on host buffers with `threads` threads."""
    import numpy as np
    from oracle import oracle as O
    c = w.cluster
    n = c.n_nodes * c.gpus_per_node
    (prod, cons), = w.phases
    total = w.data_bytes * prod.strategy.dp
    ops, loc = O.plan_data(prod, cons, c, w.data_bytes, 1)[:2]
    src = [O.data_fill(prod, c, d, True, total, 1) if O.data_shard_bytes(prod, c, d, True, total) else None
           for d in range(n)]
    dst = [np.zeros(O.data_shard_bytes(cons, c, d, False, total) // 2, np.uint16) for d in range(n)]
    delivered = sum(b * len(dsts) for (_s, dsts, _p, b) in ops + loc)
    for _ in range(warmup):
        O.data_execute(prod, cons, c, total, ops + loc, src, dst, threads)
    t0 = time.perf_counter()
    done = 0
    while True:
        O.data_execute(prod, cons, c, total, ops + loc, src, dst, threads)
        done += 1
        el = time.perf_counter() - t0
        if done >= steps and (budget_s is None or el >= budget_s or done >= 1000):
            break
    dt = (time.perf_counter() - t0) / done
    ok = all(np.array_equal(dst[d], O.data_fill(cons, c, d, False, total, 1)) for d in range(n) if dst[d].size)
    return {"gbs": delivered / dt / 1e9, "s_per_step": dt, "delivered": delivered, "correct": ok, "steps": done,
            "shard_gb": sum(x.nbytes for x in dst) / 1e9}


def cpu_sample_text(w, r: dict, threads: int) -> str:
    return (f"the whole workload ({w.description}), all phases per step, shards in host RAM "
            f"({r['shard_gb']:.1f} GB); oracle CPU reallocation (oracle/liboracle.so) with {threads} threads; "
            f"{r['delivered'] / 1e9:.2f} GB delivered per step; {r['steps']} timed steps; "
            f"checked against the oracle: {r['correct']}")


def run_reference(args) -> None:
    """--impl reference: the reference path (its CPU reallocation) on the
    box's host cores. Rank 0 only; imports nothing from the product."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    if args.config:
        print(json.dumps({"impl": "reference", "unavailable": "--config workloads: the reference arm runs the "
                                                              "named workloads of workloads.json"}), flush=True)
        return
    w = plain_workload(args.workload)
    threads = os.cpu_count() or 1
    r = cpu_realloc(w, args.steps, max(args.warmup, 1), threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(r["gbs"], 3), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": r["steps"], "warmup": args.warmup, "ms_per_step": round(r["s_per_step"] * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": workload_config(w),
        "executor": {"impl": "oracle CPU reallocation (oracle/liboracle.so: SPEC.md:541-611 restated; the "
                             "reference moves no bytes itself, SPEC.md:607)", "threads": threads},
        "host": host_info(),
        "cpu_baseline": {"value": round(r["gbs"], 3), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": cpu_sample_text(w, r, threads)},
        "e2e": {"value": round(r["gbs"], 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "verified": r["correct"],
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def load_workload(args):
    from paper_2406_14088_b200.workloads import WORKLOADS, from_config
    if args.config:
        with open(args.config) as f:
            return from_config(json.load(f), name=os.path.splitext(os.path.basename(args.config))[0])
    return WORKLOADS[args.workload]


def run_b200(args) -> None:
    import torch
    from paper_2406_14088_b200 import runtime as R
    from paper_2406_14088_b200.rlplan import BALANCED, SPEC, plan_param_realloc
    from paper_2406_14088_b200.workloads import WORKLOADS

    rank, world, local_rank = env_rank()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}; launch N>1 with torchrun")
    # More ranks than GPUs is a correctness check of the N-rank code path
    # only (two processes share a GPU and time-slice; NCCL refuses that, so
    # gloo with host tensors carries the bench's own collectives). The line
    # then says "oversubscribed" and is not a measurement.
    gpus = torch.cuda.device_count()
    oversub = world > gpus
    local_rank = local_rank % gpus
    coll = "cpu" if oversub else "cuda"
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if oversub:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    w = load_workload(args)
    if args.layers:
        from paper_2406_14088_b200.workloads import truncated
        w = truncated(w, args.layers)
    c = w.cluster()
    policy = BALANCED if args.policy == "balanced" else SPEC
    t_plan = time.perf_counter()
    plans = w.plans(policy)
    plan_ms = (time.perf_counter() - t_plan) * 1e3
    # Shard sets: phase i reads set i and writes set i+1 (round trips reuse set 0).
    names = ["train"] + [f"out{i}" for i in range(len(plans))]
    shards = {"train": (0, R.SRC)}
    bind = []
    for i, p in enumerate(plans):
        dst_name = "train" if (i == len(plans) - 1 and w.phases[i][1] == w.phases[0][0]) else f"out{i}"
        if dst_name != "train":
            shards[dst_name] = (i, R.DST)
        src_name = "train" if i == 0 else bind[-1][1]
        bind.append((src_name, dst_name))
    mode = R.PULL if args.mode == "pull" else R.PUSH
    # auto: peer stores, plus the pipelined relay where it lowers the link
    # bottleneck (single source feeding many GPUs); mc: NVLS multicast instead.
    # mc: NVLS multicast for the first phase's destinations; auto: multicast
    # sets chosen by the probe (every set a payload of which reaches every
    # GPU is allocated as multicast members and timed) or the cost model
    multicast = [bind[0][1]] if args.mode == "mc" else ("auto" if args.mode == "auto" else [])
    relay = {"auto": "auto", "relay": True}.get(args.mode, False)
    overlap = args.overlap == "on"
    # --kernel k: k for every phase (sweeps); default: per phase kind
    kernel = R.DEFAULT_KERNEL if args.kernel < 0 else args.kernel
    flag_kernel = R.DEFAULT_FLAG_KERNEL if args.kernel < 0 else args.kernel
    t_bind = time.perf_counter()
    rr = R.RankRealloc(plans, shards, bind, rank, world, local_rank, mode=mode, kernel=kernel,
                       multicast=multicast, relay=relay, overlap=overlap, flag_kernel=flag_kernel,
                       chunk_bytes=args.chunk_kib << 10, ce_min_run_bytes=-1 if args.ce == "off" else 0,
                       staged={"on": True, "off": False, "auto": "auto"}[args.staged],
                       stage_chunk_bytes=args.stage_mib << 20,
                       ce_transport={"on": True, "off": False, "auto": "auto"}[args.ce_transport],
                       probe=args.probe == "on" and world > 1)
    # executor creation only: the shard allocations inside RankRealloc are
    # timed too, so this is an upper bound of binding + descriptor upload
    bind_ms = (time.perf_counter() - t_bind) * 1e3
    stream = torch.cuda.current_stream()
    seed = 1
    for d, b in rr.buffers["train"].items():
        R.fill_shard(plans[0], R.SRC, d, b.ptr, seed)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()

    def step(ev=None):
        # Same sequence as RankRealloc.run_phase, with events around the
        # direct-copy kernel of each phase (the dominant launch).
        for i in range(len(plans)):
            if ev is not None:
                ev[i][0].record(stream)
            rr.executors[i].launch(stream, args.ctas)
            if ev is not None:
                ev[i][1].record(stream)
            if world > 1:
                rr.barrier.launch(stream)
                if rr.has_fanout[i]:
                    rr.executors[i].launch_fanout(stream, args.ctas)
                    rr.barrier.launch(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    evs = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in plans]
           for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0.record(stream)
    for k in range(args.steps):
        step(evs[k])
    t1.record(stream)
    torch.cuda.synchronize()
    clock_info = clocks.stop()
    ms = t0.elapsed_time(t1) / args.steps
    # per-step spread on this rank: step k runs from its first event to step k+1's
    starts = [evs[k][0][0] for k in range(args.steps)]
    step_ms = sorted([starts[k].elapsed_time(starts[k + 1]) for k in range(args.steps - 1)] +
                     [starts[-1].elapsed_time(t1)])
    phase_ms = [sum(evs[k][i][0].elapsed_time(evs[k][i][1]) for k in range(args.steps)) / args.steps
                for i in range(len(plans))]
    timed_out = (rr.barrier.timed_out() or rr.relay_timeouts() > 0) if world > 1 else False

    # Whole-job bytes: every rank's executor work (sum), delivered = written
    # (direct copies plus in-host fan-out); link bytes per GPU from the
    # executors' host-level accounting.
    written = sum(e.bytes_written + e.fanout_written for e in rr.executors)
    read = sum(e.bytes_read + e.fanout_read for e in rr.executors)
    # Per phase on this rank: link bytes (max of in/out) and HBM bytes of the
    # direct-copy kernel.
    P = len(plans)
    ph_wire = [max(e.wire_in, e.wire_out) for e in rr.executors]
    # HBM bytes on this GPU: everything read here (push: sources and leader
    # replicas are local) plus every store that lands here (local stores and
    # incoming peer stores); peer stores leave through the links instead.
    ph_hbm = [e.bytes_read + e.bytes_written - e.wire_out + e.wire_in for e in rr.executors]
    vals = torch.tensor([ms, written, read] + phase_ms + ph_wire + ph_hbm, dtype=torch.float64, device=coll)
    if dist:
        allv = [torch.zeros_like(vals) for _ in range(world)]
        dist.all_gather(allv, vals)
        allv = torch.stack(allv).cpu().numpy()
    else:
        allv = vals.cpu().numpy()[None, :]
    # Dominant phase: the longest direct-copy kernel over all ranks.
    ph_ms_all = allv[:, 3:3 + P]
    dom = int(ph_ms_all.max(axis=0).argmax())
    dom_ms = float(ph_ms_all[:, dom].max())
    dom_wire = float(allv[:, 3 + P + dom].max())
    dom_hbm = float(allv[:, 3 + 2 * P + dom].max())
    ms_max = float(allv[:, 0].max())
    total_written = float(allv[:, 1].sum())
    value_gbs = total_written / (ms_max * 1e-3) / 1e9

    # Verification (outside the timed region): every destination shard of every
    # phase equals the value function of its layout.
    bad = 0
    for i, (sname, dname) in enumerate(bind):
        for d, b in rr.buffers[dname].items():
            m, _ = R.verify_shard(plans[i], R.DST, d, b.ptr, seed)
            bad += m
    bad_t = torch.tensor([bad], dtype=torch.int64, device=coll)
    if dist:
        dist.all_reduce(bad_t)
    verified = int(bad_t.item()) == 0 and not timed_out

    # ---- e2e: public API with the source shards onloaded from pinned host memory.
    e2e = None
    if not args.no_e2e:
        host = {d: R.HostBuffer(b.nbytes) for d, b in rr.buffers["train"].items()}
        for d, b in rr.buffers["train"].items():
            R.memcpy_async(host[d].ptr, b.ptr, b.nbytes, 1, stream)
        res_name = bind[0][1]
        sample = 4096
        res_host = {d: R.HostBuffer(sample) for d in rr.buffers[res_name]}
        h2d = sum(b.nbytes for b in rr.buffers["train"].values())
        d2h = sample * len(res_host)
        torch.cuda.synchronize()

        copy_stream = torch.cuda.Stream()
        host_ptrs = {d: hb.ptr for d, hb in host.items()}

        def e2e_step():
            # Phase 0 onloads its sources from pinned host memory, H2D chunks
            # overlapped with the copy kernels (RankRealloc.run_phase_onload);
            # then the remaining phases as in the device-resident step.
            rr.run_phase_onload(0, host_ptrs, copy_stream, stream, args.ctas)
            for i in range(1, len(plans)):
                rr.run_phase(i, stream, args.ctas)
            for d, b in rr.buffers[res_name].items():
                R.memcpy_async(res_host[d].ptr, b.ptr, min(sample, b.nbytes), 1, stream)
            R.stream_sync(stream)

        e2e_step()
        if dist:
            dist.barrier()
        e0 = time.perf_counter()
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        for _ in range(e2e_steps):
            e2e_step()
        e_ms = (time.perf_counter() - e0) * 1e3 / e2e_steps
        # the onloaded (pipelined) path must produce the same shards
        e2e_bad = 0
        for i, (sname, dname) in enumerate(bind):
            for d, b in rr.buffers[dname].items():
                e2e_bad += R.verify_shard(plans[i], R.DST, d, b.ptr, seed)[0]
        ev = torch.tensor([e_ms, h2d, d2h, e2e_bad], dtype=torch.float64, device=coll)
        if dist:
            mx = ev.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            sm = ev.clone()
            dist.all_reduce(sm)
            e_ms, h2d, d2h, e2e_bad = float(mx[0]), float(sm[1]), float(sm[2]), float(sm[3])
        else:
            e_ms, h2d, d2h, e2e_bad = float(ev[0]), float(ev[1]), float(ev[2]), float(ev[3])
        verified = verified and e2e_bad == 0
        e2e = {"value": round(total_written / (e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e_ms, 3),
               "timing": "host wall clock around stream-synchronised steps, max over ranks",
               "path": "public API: RankRealloc.run_phase_onload (H2D chunks pipelined with the copy kernels)",
               "results": "the resharded weights stay in HBM for the engine that uses them next (generation / "
                          "training); d2h reads back a 4 KiB sample of every destination shard per step. Copying "
                          "every result to the host would bound e2e by the same host link as the onload",
               "verified": e2e_bad == 0}
        for hb in list(host.values()) + list(res_host.values()):
            hb.free()

    cpu = None
    oracle_checked, oracle_bad = False, None
    if rank == 0 and world == 1 and not args.no_cpu and not args.config and not args.layers:
        # the reference path on this box's host cores, same workload (plain
        # objects from workloads.json), after the GPU arm has released its
        # pinned host buffers
        threads = os.cpu_count() or 1
        pw = plain_workload(w.name)
        # the oracle as the checker of the GPU arm: every byte of every
        # destination shard of every phase against its expected shard
        oracle_bad = oracle_check(rr, bind, plans, pw, seed, threads)
        oracle_checked = True
        verified = verified and oracle_bad == 0
        try:
            r = cpu_realloc(pw, 1, 1, threads, budget_s=args.cpu_budget)
            cpu = {"value": round(r["gbs"], 3), "unit": "GB/s", "cores": threads, "kind": "port",
                   "sample": cpu_sample_text(pw, r, threads)}
        except MemoryError as e:
            cpu = {"value": None, "unit": "GB/s", "cores": threads, "kind": "port", "sample": f"not run: {e}"}

    if rank == 0:
        peaks = measured_peaks()
        # the kernels the library chose for the dominant phase's direct copies
        _ldst, bulk = rr.executors[dom].phase_kernels(0)
        kname = "rr_bulk_kernel" if bulk else "rr_copy_kernel"
        if world == 1:
            achieved = dom_hbm / (dom_ms * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": profile_traffic(w.name),
                    "traffic_source": (f"profiles/{w.name}.ncu.json: dram__bytes_read+write of this kernel per "
                                       "launch from a committed ncu --set full capture, not measured in this run"),
                    "kernel": kname, "phase": dom, "peak_source": peaks["source"],
                    "algorithmic_bytes_per_launch": int(dom_hbm)}
        else:
            # The dominant phase is bound by the links or, when in-host
            # fan-outs run inside it (overlap), by HBM: report the resource it
            # uses the larger fraction of, with the other beside it.
            hbm_achieved = dom_hbm / (dom_ms * 1e-3) / 1e9
            hbm_roof = {"bound": "hbm", "achieved": round(hbm_achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": round(hbm_achieved / peaks["hbm_gbs"], 4),
                        "algorithmic_bytes_per_launch": int(dom_hbm), "peak_source": peaks["source"]}
            # bottleneck GPU's link bytes over the slowest rank's kernel time
            achieved = dom_wire / (dom_ms * 1e-3) / 1e9
            # ncu: NVLink protocol adds 18.75% to the payload bytes on the wire
            # (profiles/r01_nvlink_counters_n2.json: 9535619072 / 8029995008)
            proto = 9535619072 / 8029995008
            roof = {"bound": "nvlink", "achieved": round(achieved, 1), "peak": NVLINK_PEAK, "unit": "GB/s",
                    "frac": round(achieved / NVLINK_PEAK, 4), "traffic": int(dom_wire * proto),
                    "traffic_source": "payload x measured NVLink protocol factor (ncu nvltx__bytes)",
                    "wire_frac_incl_protocol": round(achieved * proto / NVLINK_PEAK, 4), "kernel": kname,
                    "phase": dom, "peak_source": "nominal NVLink 5 per direction (measured ceilings: SM peer stores "
                                                               "~710, one copy-engine copy ~780 GB/s; "
                                                               "profiles/r01_nvlink_probe_n2.txt)",
                    "algorithmic_bytes_per_launch": int(dom_wire)}
            if (dom in rr.staged_phases or dom in rr.ce_phases or dom in rr.nccl_phases
                    or rr.executors[dom].ce_runs()[0] > 0):
                # copy engines carry (most of) this phase's link bytes: the SM
                # stores' protocol factor does not apply to them
                roof.update({"traffic": None, "wire_frac_incl_protocol": None,
                             "traffic_source": "copy-engine / NCCL transfers: no per-kernel ncu counter",
                             "kernel": ("copy engines (staged gather) + " if dom in rr.staged_phases
                                   else "copy-engine transport + " if dom in rr.ce_phases
                                   else "NCCL + " if dom in rr.nccl_phases
                                   else "copy-engine runs + ") + kname})
            if hbm_roof["frac"] > roof["frac"]:
                hbm_roof.update({"traffic": None, "kernel": kname, "phase": dom,
                                 "per_gpu": "max over ranks of this GPU's reads + stores landing in its HBM",
                                 "peak_note": "peak is the 1:1 copy figure; this phase is write-heavy and pure "
                                              "writes reach 7622 GB/s on B200 (profiles/r01_hbm_mix_probe.txt), "
                                              "so frac can exceed 1",
                                 "nvlink": {k: roof[k] for k in ("achieved", "peak", "frac", "wire_frac_incl_protocol",
                                                                  "algorithmic_bytes_per_launch")}})
                roof = hbm_roof
            else:
                roof["hbm"] = {k: hbm_roof[k] for k in ("achieved", "peak", "frac", "algorithmic_bytes_per_launch")}
        nvl = float(allv[:, 3 + P:3 + 2 * P].sum(axis=1).max() / (ms_max * 1e-3) / 1e9) if world > 1 else 0.0
        line = {
            "metric": METRIC, "value": round(value_gbs, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max, 4), "higher_is_better": True, "scaling": "strong",
            "scaling_note": ("total work fixed (the workload's plan devices spread over N GPUs): at N=1 every "
                             "move is a local HBM relayout, at N>1 each GPU must also receive the slices held "
                             "on other GPUs over NVLink (900 GB/s per direction vs ~6.5 TB/s HBM), so time "
                             "need not fall with N; compare each N against its own roofline"),
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": (workload_config(plain_workload(w.name)) if not (args.config or args.layers)
                       else workload_config(w)),
            "executor": {"plan_devices_per_gpu": w.devices // world, "policy": args.policy, "mode": args.mode,
                         "multicast_sets": rr.multicast, "relay_phases": rr.relay_phases,
                         "overlap_phases": rr.overlap_phases, "copy_kernel": kname,
                         "ce_runs": [list(e.ce_runs()) for e in rr.executors], "staged_phases": rr.staged_phases,
                         "ce_transport_phases": rr.ce_phases, "nccl_phases": rr.nccl_phases,
                         "ce_transport_estimates_ms": {pi: [round(x * 1e3, 3) for x in v]
                                                       for pi, v in rr.ce_estimates.items()},
                         "bulk_variants": {"plain": 1 if kernel is None else kernel, "flag_synchronised": flag_kernel},
                         "chunk_kib": args.chunk_kib or "library default (256; smaller for phases too small for it)",
                         "ctas": args.ctas or "resident capacity",
                         "policy_probe": getattr(rr, "probe_log", None)},
            "host": host_info(),
            "phase_ms": [round(float(x), 4) for x in ph_ms_all.max(axis=0)],
            "step_ms": {"median": round(step_ms[len(step_ms) // 2], 4), "best": round(step_ms[0], 4),
                        "worst": round(step_ms[-1], 4), "of": "rank 0's timed steps (CUDA events)"},
            "nvlink_gbs_per_gpu": round(nvl, 2),
            # per rank: its link bytes (max of in / out, summed over phases) over the
            # step, and per phase over that phase's kernel time (the slowest rank's)
            "nvlink_gbs_per_rank": ([round(float(x) / (ms_max * 1e-3) / 1e9, 2)
                                     for x in allv[:, 3 + P:3 + 2 * P].sum(axis=1)] if world > 1 else None),
            "nvlink_gbs_per_rank_phase": ([[round(float(allv[r, 3 + P + i]) / (max(float(ph_ms_all[:, i].max()), 1e-6) * 1e-3) / 1e9, 1)
                                            for i in range(P)] for r in range(world)] if world > 1 else None),
            "bytes_per_step": int(total_written),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            # this rank's kernels in the timed region: copy kernels of every
            # phase, plus the barrier(s) and the fan-out kernels when N > 1
            # (copy-engine copies and their stream-written flags are not kernels)
            "gpu_launches": args.steps * sum(
                e.kernel_count()[0] + ((1 + rr.has_fanout[i] * (1 + e.kernel_count()[1])) if world > 1 else 0)
                for i, e in enumerate(rr.executors)),
            "copy_engine_submissions": args.steps * sum(e.ce_runs()[0] + e.stage_pushes()[0] for e in rr.executors),
            "clocks": clock_info,
            # host side, once per plan (not in the timed region): planning +
            # lowering, and rank 0's buffer allocation + executor binding/upload
            "host_ms": {"plan_and_lower": round(plan_ms, 3), "allocate_and_bind": round(bind_ms, 1)},
            "verified": verified,
            "verified_by": ("device regenerate-and-compare of every destination shard (product fill function)"
                            + ("; and every byte of every destination shard against the oracle's expected shards "
                               f"(oracle/liboracle.so orc_check_range, in the cpu_baseline leg): "
                               f"{'0' if not oracle_bad else oracle_bad} mismatching elements"
                               if oracle_checked else "")),
        }
        if oversub:
            line["oversubscribed"] = f"{world} ranks on {gpus} GPUs: correctness run, not a measurement"
        print(json.dumps(line), flush=True)
    rr.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def oracle_check(rr, bind, plans, pw, seed: int, threads: int) -> int:
    """Compare every destination shard the GPU arm wrote with the oracle's
    expected shard (streamed 256 MiB windows, D2H of window k + 1 overlapped
    with the check of window k). Returns the mismatching elements."""
    from oracle import oracle as O
    from paper_2406_14088_b200 import runtime as R
    window = 256 << 20
    hosts = [R.HostBuffer(window), R.HostBuffer(window)]
    bad = 0
    try:
        for i, (_sname, dname) in enumerate(bind):
            dst = pw.phases[i][1]
            for d, b in sorted(rr.buffers[dname].items()):
                offs = list(range(0, b.nbytes, window))
                if offs:
                    R.memcpy_async(hosts[0].ptr, b.ptr, min(window, b.nbytes), 1)
                for k, off in enumerate(offs):
                    R.stream_sync()
                    if k + 1 < len(offs):
                        R.memcpy_async(hosts[(k + 1) % 2].ptr, b.ptr + offs[k + 1],
                                       min(window, b.nbytes - offs[k + 1]), 1)
                    bad += O.check_range(pw.model, dst, pw.cluster, d, seed, off, min(window, b.nbytes - off),
                                         hosts[k % 2].ptr, threads)[0]
                R.stream_sync()
    finally:
        for h in hosts:
            h.free()
    return bad


def profile_traffic(workload: str):
    """dram__bytes_read+write per launch of the dominant kernel from the
    committed ncu summary (profiles/<workload>.ncu.json), if any."""
    path = os.path.join(ROOT, "profiles", f"{workload}.ncu.json")
    try:
        with open(path) as f:
            return json.load(f).get("traffic_bytes_per_launch")
    except Exception:
        return None


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", default="llama7b_tp8_dp8_roundtrip")
    ap.add_argument("--config", default=None,
                    help="realloc-plan/data-plan config JSON (cli.py format, plus \"back\": true) instead of "
                         "a named workload")
    ap.add_argument("--policy", choices=["balanced", "spec"], default="balanced")
    ap.add_argument("--mode", choices=["auto", "push", "pull", "mc", "relay"], default="auto",
                    help="push = SM peer stores; relay = push + pipelined relay for payloads reaching >= 2 "
                         "other GPUs; mc = push + NVLS multicast for the first phase's destination (N > 1); "
                         "auto = push, relay where it lowers the link bottleneck")
    ap.add_argument("--ce", choices=["on", "off"], default="on",
                    help="copy-engine runs for >= 256 MiB ranges laid out identically in a source and a remote "
                         "destination shard (push mode; library default)")
    ap.add_argument("--ce-transport", choices=["auto", "on", "off"], default="auto",
                    help="copy-engine transport of remote pieces (2D/3D copies merged across layers, rotation "
                         "rounds, straight into the destination shards); auto = phases without in-host fan-out "
                         "where the measured rates predict >= 5%% less link time than SM peer stores")
    ap.add_argument("--probe", choices=["on", "off"], default="on",
                    help="N > 1: choose each phase's delivery scheme by timing every scheme the switches allow on "
                         "the real buffers at bind time (max over ranks; executor.policy_probe) instead of the "
                         "cost model alone")
    ap.add_argument("--staged", choices=["auto", "on", "off"], default="auto",
                    help="staged gather for phases that read other GPUs' sources: whole source shards pushed by "
                         "copy engines in rotation rounds, unpacked per 512 MiB piece; auto = from 4 GPUs on, "
                         "all-gather-shaped phases")
    ap.add_argument("--stage-mib", type=int, default=512, help="staged-gather piece size (MiB)")
    ap.add_argument("--overlap", choices=["on", "off"], default="on",
                    help="run in-host fan-outs per chunk inside the first phase (N > 1) instead of after a barrier")
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--chunk-kib", type=int, default=0, help="work-item size in KiB (0 = library default)")
    ap.add_argument("--layers", type=int, default=0, help="truncate the model (profiling only)")
    ap.add_argument("--kernel", type=int, default=-1, help="copy engine: 0 LDG/STG, 1..5 TMA bulk (-1 default)")
    ap.add_argument("--cpu-budget", type=float, default=10.0,
                    help="seconds of timed CPU reallocation in the cpu_baseline leg (whole workload, >= 1 step)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
