"""Multi-process GPU parity worker (launched by tests/test_multigpu.py via
torchrun, one process per GPU — or several per GPU, oversubscribed). Each
rank hosts a contiguous block of the 8 plan devices; destination shards of
remote ranks are reached through CUDA IPC and written by peer stores (NVLink
between GPUs; the same IPC mappings within one GPU when oversubscribed).
Every rank compares its hosted destination shards with the CPU oracle and
the results are all-reduced.

Rank 0 prints one line per case: `case <name>: ok|FAIL <seconds>`.
Environment: RR_FUZZ_CASES (24), RR_FUZZ_SEED (2406), RR_FULL_7B=1 (full-size
7B round trip, every byte against the oracle; distinct GPUs only)."""
from __future__ import annotations

import contextlib
import dataclasses
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from _helpers import oracle_compare_device, placement, random_placement  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2406_14088_b200 import runtime as R  # noqa: E402
from paper_2406_14088_b200.rlplan import (BALANCED, MODELS, DeviceMesh, ParallelStrategy, Placement,  # noqa: E402
                                          b200_cluster, plan_param_realloc)
from paper_2406_14088_b200.workloads import WORKLOADS  # noqa: E402

TINY_GQA = dataclasses.replace(MODELS["tiny"], name="tiny_gqa", hidden_size=512, num_attention_heads=16,
                               num_kv_heads=8, intermediate_size=1024)
TINY_MQA = dataclasses.replace(TINY_GQA, name="tiny_mqa", num_attention_heads=8, num_kv_heads=1, num_layers=3)
SPECIAL = O.SEED_SPECIAL  # special-value bf16 words (zeros, infinities, NaN payloads, subnormals, any pattern)

CASES = [
    ((1, 1, 8, 0, 0), (1, 8, 1, 0, 0)),   # tp8 -> dp8 all-gather
    ((4, 1, 2, 2, 1), (1, 1, 8, 1, 1)),   # 34B-style grouped/concat reinterleave
    ((2, 1, 4, 0, 0), (1, 1, 8, 0, 0)),   # 70B-style pp2 tp4 -> tp8
    ((2, 1, 4, 0, 0), (1, 2, 4, 0, 0)),   # 13B-style stage remap
    ((1, 8, 1, 2, 1), (4, 1, 2, 0, 0)),   # dp8 replicas -> pp4 tp2
]
REPLICATE = (Placement(DeviceMesh(0, 1, 0, 1), ParallelStrategy()), placement(8, 1, 8, 1))


def pl(spec):
    return placement(8, *spec[:3], qkv=spec[3], gate_up=spec[4])


PAGE = 2 << 20  # rr_device_alloc pads every allocation to whole 2 MiB pages
GUARD = 0xA5


def guard_tails(bufs):
    """compute-sanitizer is closed on this pool: out-of-bounds stores are
    caught instead by a known pattern in the padding after every local
    shard (up to 64 KiB of it), checked after each launch."""
    from paper_2406_14088_b200._lib import check, lib
    out = []
    for b in bufs:
        if not isinstance(b, R.DeviceBuffer):
            continue
        start = max(b.nbytes, 256)
        tail = min((max(b.nbytes, 256) + PAGE - 1) // PAGE * PAGE - start, 64 << 10)
        if tail > 0:
            check(lib.rr_memset(b.ptr + start, GUARD, tail, None))
            out.append((b, start, tail))
    return out


def tails_intact(guards) -> bool:
    from paper_2406_14088_b200._lib import check, lib
    for b, start, tail in guards:
        h = np.empty(tail, np.uint8)
        check(lib.rr_memcpy(h.ctypes.data, b.ptr + start, tail, 1, None, 1))
        if not (h == GUARD).all():
            return False
    return True


class Worker:
    def __init__(self):
        self.rank, self.world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
        # More ranks than GPUs (world 2/4 on one GPU, world 8 on four): ranks
        # share a GPU and their kernels time-slice; IPC, flags, copy engines
        # and barriers behave as across GPUs. NCCL refuses two ranks per GPU,
        # so gloo carries the host-side collectives; multicast needs distinct
        # GPUs and is skipped.
        gpus = torch.cuda.device_count()
        self.local = int(os.environ["LOCAL_RANK"]) % gpus
        self.oversub = self.world > gpus
        torch.cuda.set_device(self.local)
        if self.oversub:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
        self.c = b200_cluster(8)
        # RR_QUICK=1 (the 1-GPU oversubscribed pytest): one copy kernel per
        # scheme where the full run sweeps both; every scheme still runs
        self.quick = os.environ.get("RR_QUICK") == "1"
        self.kernels = (1,) if self.quick else (1, 0)
        self.failures: list = []
        self.ce_runs = 0        # copy-engine runs issued by this rank
        self.staged_phases = 0  # staged-gather phases set up

    @contextlib.contextmanager
    def case(self, label: str):
        n0, t0 = len(self.failures), time.time()
        try:
            yield
        except Exception as e:  # a crash in one case is a failure, the others still run
            self.failures.append(f"{label}: {type(e).__name__}: {e}")
        if self.rank == 0:
            ok = "ok" if len(self.failures) == n0 else "FAIL"
            print(f"case {label}: {ok} {time.time() - t0:.2f}s", flush=True)

    def run(self, label, model, src, dst, seed, reps=1, policy=BALANCED, onload_chunk=0, zero_between=True,
            **kw):
        """Plan src -> dst, bind RankRealloc with `kw`, launch phase 0 `reps`
        times (epochs advance per launch), each time comparing every hosted
        destination byte with the oracle; flag and barrier timeouts fail."""
        with self.case(label):
            plan = plan_param_realloc(model, src, dst, self.c, policy)
            rr = R.RankRealloc([plan], {"a": (0, R.SRC), "b": (0, R.DST)}, [("a", "b")], self.rank, self.world,
                               self.local, **kw)
            try:
                self.ce_runs += sum(e.ce_runs()[0] for e in rr.executors)
                self.staged_phases += len(rr.staged_phases)
                for d, b in rr.buffers["a"].items():
                    R.fill_shard(plan, R.SRC, d, b.ptr, seed)
                for rep in range(reps):
                    if zero_between:
                        for b in rr.buffers["b"].values():
                            b.zero()
                    guards = guard_tails(list(rr.buffers["a"].values()) + list(rr.buffers["b"].values()))
                    torch.cuda.synchronize()
                    dist.barrier()
                    hosts = None
                    if onload_chunk and rep % 2 == 1:  # odd reps: sources onloaded from pinned host memory
                        hosts = {d: R.HostBuffer(b.nbytes) for d, b in rr.buffers["a"].items()}
                        for d, hb in hosts.items():
                            hb.array()[:] = rr.buffers["a"][d].to_host()
                        rr.run_phase_onload(0, {d: hb.ptr for d, hb in hosts.items()}, torch.cuda.Stream(),
                                            chunk_bytes=onload_chunk)
                    else:
                        rr.run_phase(0)
                    torch.cuda.synchronize()
                    for d, b in rr.buffers["b"].items():
                        got = b.to_host()
                        want = O.fill(model, dst, self.c, d, seed)
                        if not np.array_equal(got, want):
                            self.failures.append(f"{label} rep {rep}: device {d} differs in "
                                                 f"{int(np.count_nonzero(got != want))} elements")
                    dist.barrier()  # every rank's stores are done before the guards are read
                    if not tails_intact(guards):
                        self.failures.append(f"{label} rep {rep}: a store landed past the end of a shard")
                    for hb in (hosts or {}).values():
                        hb.free()
                if rr.relay_timeouts() or rr.barrier.timed_out():
                    self.failures.append(f"{label}: flag or barrier timeouts")
                dist.barrier()
            finally:
                rr.close()

    # ---- sections ---------------------------------------------------------

    def basic(self):
        """Peer stores / peer loads, flat and hierarchical, both kernels."""
        for mode in (R.PUSH, R.PULL):
            for kernel in self.kernels:
                for hier in (True, False):
                    for sp, dp in CASES:
                        seed = 21 if hier else SPECIAL | 21
                        self.run(f"basic {sp}->{dp} mode={mode} kernel={kernel} hier={hier} seed={seed:#x}",
                                 TINY_GQA, pl(sp), pl(dp), seed, mode=mode, kernel=kernel, hierarchical=hier)

    def multicast(self):
        """NVLS multicast (K3): one store through multimem.st reaches every GPU."""
        if self.oversub or not R.multicast_supported(self.local):
            if self.rank == 0:
                print("dist_worker: NVLS multicast not supported or GPUs shared, skipped", flush=True)
            return
        for src, dst in (REPLICATE, (pl((1, 1, 8, 0, 0)), pl((1, 8, 1, 0, 0)))):
            for seed in (23, SPECIAL | 23):
                self.run(f"multicast {src.strategy}->{dst.strategy} seed={seed:#x}", TINY_GQA, src, dst, seed,
                         multicast=["b"])
            # multicast members allocated for the probe: the probe times
            # multicast beside every other scheme (peers reach the members by
            # mapped physical memory), and a non-multicast scheme on them
            self.run(f"multicast-probe {src.strategy}->{dst.strategy}", TINY_GQA, src, dst, SPECIAL | 24, reps=2,
                     multicast="auto", probe=True, overlap=True, relay="auto", staged=True, ce_transport=True)
            with self.case(f"peer stores into multicast members {src.strategy}->{dst.strategy}"):
                plan = plan_param_realloc(TINY_GQA, src, dst, self.c, BALANCED)
                rr = R.RankRealloc([plan], {"a": (0, R.SRC), "b": (0, R.DST)}, [("a", "b")], self.rank,
                                   self.world, self.local, multicast="auto", probe=True, overlap=True)
                try:
                    for sc in (R.Scheme(overlap=True), R.Scheme(ce_transport=True, overlap=True)):
                        rr._unbind_phase(0)
                        rr.schemes[0] = sc
                        rr._bind_phase(0, sc)
                        rr.executors = [b.executor for b in rr.bindings]
                        for d, b in rr.buffers["a"].items():
                            R.fill_shard(plan, R.SRC, d, b.ptr, SPECIAL | 25)
                        for b in rr.buffers["b"].values():
                            b.zero()
                        torch.cuda.synchronize()
                        dist.barrier()
                        rr.run_phase(0)
                        torch.cuda.synchronize()
                        for d, b in rr.buffers["b"].items():
                            if not np.array_equal(b.to_host(), O.fill(TINY_GQA, dst, self.c, d, SPECIAL | 25)):
                                self.failures.append(f"{sc.label()} into multicast members: device {d} differs")
                        dist.barrier()
                finally:
                    rr.close()

    def overlap(self):
        """Overlapped in-host fan-out (star flags), with and without the relay."""
        for relay, kernel in [(r, k) for k in self.kernels for r in (False, True)]:
            for sp, dp in CASES:
                seed = SPECIAL | 37 if kernel else 37
                self.run(f"overlap relay={relay} kernel={kernel} {sp}->{dp} seed={seed:#x}", TINY_GQA, pl(sp),
                         pl(dp), seed, reps=2, relay=relay, overlap=True, kernel=kernel, flag_kernel=kernel)

    def relay(self):
        """Pipelined relay: chunks travel source -> GPU -> GPU with per-chunk flags."""
        cases = [REPLICATE, (pl((1, 1, 8, 0, 0)), pl((1, 8, 1, 0, 0))),
                 (placement(2, 1, 1, 2, offset=2), placement(8, 1, 4, 2))]
        for src, dst in cases:
            for kernel in self.kernels:
                seed = SPECIAL | 29 if kernel else 29
                self.run(f"relay kernel={kernel} {src.strategy}->{dst.strategy} seed={seed:#x}", TINY_GQA, src, dst,
                         seed, reps=3, relay=True, kernel=kernel, flag_kernel=kernel)
                # the same chains on copy engines (hop-by-hop pieces, stream
                # wait/write flags), plain and onloaded, with and without star
                for overlap in (False, True):
                    self.run(f"ce-relay kernel={kernel} overlap={overlap} {src.strategy}->{dst.strategy} (+onload)",
                             TINY_GQA, src, dst, SPECIAL | 30, reps=3, onload_chunk=32 << 10, relay=True,
                             ce_transport=True, overlap=overlap, kernel=kernel, flag_kernel=kernel)

    def ce_runs_cases(self):
        """Copy-engine runs on stage remaps (forced down to 4 KiB ranges so the
        tiny model has some), hierarchical and flat, plain and onloaded."""
        for sp, dp in (((2, 1, 4, 0, 0), (1, 2, 4, 0, 0)), ((2, 2, 2, 1, 1), (1, 4, 2, 1, 1)),
                       ((1, 2, 4, 2, 1), (2, 1, 4, 2, 1))):
            for hier in (True, False):
                self.run(f"ce-runs {sp}->{dp} hier={hier} (+onload)", TINY_GQA, pl(sp), pl(dp), SPECIAL | 77,
                         reps=2, onload_chunk=64 << 10, hierarchical=hier, ce_min_run_bytes=4096)

    def ce_transport(self):
        """Copy-engine transport: remote pieces by copy engine as 2D / 3D copies
        merged across layers, in rotation rounds, plain and onloaded, with the
        fan-out phase after it where a host holds several destinations."""
        m = dataclasses.replace(TINY_GQA, num_layers=6)
        for sp, dp in CASES:
            for star in (False, True):  # star: fan-out inside phase 0 on per-copy flags
                for kernel in (self.kernels if star else (1,)):
                    self.run(f"ce-transport {sp}->{dp} star={star} kernel={kernel} (+onload)", m, pl(sp), pl(dp),
                             SPECIAL | 83, reps=3, onload_chunk=32 << 10, ce_transport=True, overlap=star,
                             kernel=kernel, flag_kernel=kernel)
        # hybrid: unmerged row-parallel pieces on SM stores beside the copy engines
        for sp, dp in CASES[1:3]:
            src, dst = pl(sp), pl(dp)
            label = f"ce-transport hybrid {sp}->{dp}"
            with self.case(label):
                plan = plan_param_realloc(m, src, dst, self.c, BALANCED)
                rr = R.RankRealloc([plan], {"a": (0, R.SRC), "b": (0, R.DST)}, [("a", "b")], self.rank,
                                   self.world, self.local, ce_transport=True)
                try:
                    rr._unbind_phase(0)
                    rr.schemes[0] = R.Scheme(ce_transport=True, ce_hybrid=True)
                    rr._bind_phase(0, rr.schemes[0])
                    rr.executors = [b.executor for b in rr.bindings]
                    for d, b in rr.buffers["a"].items():
                        R.fill_shard(plan, R.SRC, d, b.ptr, SPECIAL | 85)
                    torch.cuda.synchronize()
                    dist.barrier()
                    rr.run_phase(0)
                    torch.cuda.synchronize()
                    for d, b in rr.buffers["b"].items():
                        if not np.array_equal(b.to_host(), O.fill(m, dst, self.c, d, SPECIAL | 85)):
                            self.failures.append(f"{label}: device {d} differs")
                    dist.barrier()
                finally:
                    rr.close()
        # replicate (one source, fan-out on every GPU)
        self.run("ce-transport replicate star=True", m, REPLICATE[0], REPLICATE[1], SPECIAL | 84, reps=2,
                 ce_transport=True, overlap=True)

    def probe(self):
        """Bind-time probe: every scheme the switches allow is timed on the real
        buffers (max over ranks) and the fastest kept; the chosen executor
        must be bit-exact like any other, and every rank must agree."""
        m = dataclasses.replace(TINY_GQA, num_layers=6)
        for sp, dp in CASES[:3] + [((1, 1, 1, 0, 0), (1, 8, 1, 0, 0))]:
            src = REPLICATE[0] if sp == (1, 1, 1, 0, 0) else pl(sp)
            label = f"probe {sp}->{dp}"
            with self.case(label):
                plan = plan_param_realloc(m, src, pl(dp), self.c, BALANCED)
                rr = R.RankRealloc([plan], {"a": (0, R.SRC), "b": (0, R.DST)}, [("a", "b")], self.rank, self.world,
                                   self.local, relay="auto", overlap=True, staged=True, ce_transport=True,
                                   stage_chunk_bytes=64 << 10, probe=True)
                try:
                    log = self._agree(rr.probe_log)
                    if self.world > 1 and not log:
                        self.failures.append(f"{label}: no probe ran")
                    if self.rank == 0:
                        print(f"  {label}: {log}", flush=True)
                    for d, b in rr.buffers["a"].items():
                        R.fill_shard(plan, R.SRC, d, b.ptr, SPECIAL | 61)
                    for _rep in range(2):
                        for b in rr.buffers["b"].values():
                            b.zero()
                        torch.cuda.synchronize()
                        dist.barrier()
                        rr.run_phase(0)
                        torch.cuda.synchronize()
                        for d, b in rr.buffers["b"].items():
                            if not np.array_equal(b.to_host(), O.fill(m, pl(dp), self.c, d, SPECIAL | 61)):
                                self.failures.append(f"{label}: device {d} differs")
                    if rr.relay_timeouts() or rr.barrier.timed_out():
                        self.failures.append(f"{label}: flag or barrier timeouts")
                    dist.barrier()
                finally:
                    rr.close()

    def nccl_scheme(self):
        """Scheme(nccl=True), the library baseline the probe times: whole
        source shards by NCCL (broadcast for a lone source, else send/recv),
        then a local pull unpack; plain and onloaded."""
        if self.oversub:
            return
        m = dataclasses.replace(TINY_GQA, num_layers=6)
        for src, dst in [(pl(a), pl(b)) for a, b in CASES] + [REPLICATE]:
            label = f"nccl-scheme {src.strategy}->{dst.strategy}"
            with self.case(label):
                plan = plan_param_realloc(m, src, dst, self.c, BALANCED)
                rr = R.RankRealloc([plan], {"a": (0, R.SRC), "b": (0, R.DST)}, [("a", "b")], self.rank, self.world,
                                   self.local)
                try:
                    rr._unbind_phase(0)
                    rr.schemes[0] = R.Scheme(nccl=True)
                    rr._bind_phase(0, rr.schemes[0])
                    rr.executors = [b.executor for b in rr.bindings]
                    seed = SPECIAL | 87
                    for d, b in rr.buffers["a"].items():
                        R.fill_shard(plan, R.SRC, d, b.ptr, seed)
                    for rep in range(2):
                        for b in rr.buffers["b"].values():
                            b.zero()
                        torch.cuda.synchronize()
                        dist.barrier()
                        hosts = None
                        if rep == 1:
                            hosts = {d: R.HostBuffer(b.nbytes) for d, b in rr.buffers["a"].items()}
                            for d, hb in hosts.items():
                                hb.array()[:] = rr.buffers["a"][d].to_host()
                            rr.run_phase_onload(0, {d: hb.ptr for d, hb in hosts.items()}, torch.cuda.Stream())
                        else:
                            rr.run_phase(0)
                        torch.cuda.synchronize()
                        for d, b in rr.buffers["b"].items():
                            if not np.array_equal(b.to_host(), O.fill(m, dst, self.c, d, seed)):
                                self.failures.append(f"{label} rep {rep}: device {d} differs")
                        for hb in (hosts or {}).values():
                            hb.free()
                    dist.barrier()
                finally:
                    rr.close()

    def _agree(self, obj):
        out = [None] * self.world
        dist.all_gather_object(out, [e["chosen"] for e in obj])
        if any(o != out[0] for o in out):
            self.failures.append(f"ranks chose different schemes: {out}")
        return obj

    def staged(self):
        """Staged gather (copy-engine rotation + per-piece unpack), small pieces,
        both unpack kernels, plain / onloaded / plain again (flag epochs)."""
        for sp, dp in (((1, 1, 8, 0, 0), (1, 8, 1, 0, 0)), ((2, 1, 4, 1, 1), (1, 1, 8, 0, 0)),
                       ((1, 2, 4, 0, 0), (4, 1, 2, 2, 1)), ((1, 8, 1, 0, 0), (1, 1, 8, 0, 0))):
            for kernel in self.kernels:
                self.run(f"staged {sp}->{dp} kernel={kernel} (+onload)", TINY_GQA, pl(sp), pl(dp), SPECIAL | 91,
                         reps=3, onload_chunk=64 << 10, staged=True, stage_chunk_bytes=64 << 10, kernel=kernel,
                         flag_kernel=kernel)

    def staged_many_items(self):
        """A staged unpack with far more items than resident CTAs (one CTA per
        SM, 1 KiB items): the unpack spins on piece flags while the senders'
        copy streams raise them (no kernel takes part in signalling)."""
        self.run("staged many-items tp8->dp8 chunk=1KiB", TINY_GQA, pl((1, 1, 8, 0, 0)), pl((1, 8, 1, 0, 0)),
                 SPECIAL | 93, reps=2, staged=True, stage_chunk_bytes=16 << 10, chunk_bytes=1024, kernel=0,
                 flag_kernel=0)

    def fuzz(self):
        """Random placement pairs with random delivery options (same seed on
        every rank, so all ranks build the same plans and executors)."""
        rng = random.Random(int(os.environ.get("RR_FUZZ_SEED", "2406")))
        for i in range(int(os.environ.get("RR_FUZZ_CASES", "24"))):
            fm = (TINY_GQA, TINY_MQA)[i % 2]
            src, dst = random_placement(rng, fm), random_placement(rng, fm)
            kw = dict(mode=rng.choice([R.PUSH, R.PULL]), hierarchical=rng.random() < 0.7,
                      relay=rng.choice([False, True, "auto"]), overlap=rng.random() < 0.5,
                      chunk_bytes=rng.choice([0, 8192, 65536]),
                      ce_min_run_bytes=rng.choice([-1, 0, 4096]),  # off, default (256 MiB: none here), >= 4 KiB
                      staged=rng.random() < 0.25, stage_chunk_bytes=32 << 10,
                      ce_transport=rng.random() < 0.3,
                      probe=rng.random() < 0.15)  # bind-time probe: every allowed scheme, fastest kept
            kw["kernel"] = kw["flag_kernel"] = rng.choice([0, 1, 5])
            policy = rng.choice([0, 1])
            seed = (SPECIAL if i % 3 == 0 else 0) | (50 + i)
            opts = " ".join(f"{k}={v}" for k, v in kw.items() if k != "flag_kernel")
            self.run(f"fuzz {i} {src.strategy}{src.mesh}->{dst.strategy}{dst.mesh} policy={policy} {opts}", fm,
                     src, dst, seed, reps=2, policy=policy, **kw)

    def full_7b(self):
        """BASELINE configs[1] at full size across the GPUs: every byte of
        every hosted shard against the oracle (streamed windows)."""
        if os.environ.get("RR_FULL_7B") != "1" or self.oversub:
            return
        with self.case("full-size 7B tp8->dp8->tp8 (every byte vs oracle)"):
            w = WORKLOADS["llama7b_tp8_dp8_roundtrip"]
            (train, gen), _ = w.phases
            plans = [plan_param_realloc(w.model, s, d, self.c, BALANCED) for (s, d) in w.phases]
            rr = R.RankRealloc(plans, {"train": (0, R.SRC), "gen": (0, R.DST)},
                               [("train", "gen"), ("gen", "train")], self.rank, self.world, self.local,
                               overlap=True, staged="auto")
            try:
                seed = SPECIAL | 4
                for d, b in rr.buffers["train"].items():
                    R.fill_shard(plans[0], R.SRC, d, b.ptr, seed)
                torch.cuda.synchronize()
                dist.barrier()
                for _ in range(2):
                    rr.run_phase(0)
                    rr.run_phase(1)
                torch.cuda.synchronize()
                for name, p in (("gen", gen), ("train", train)):
                    for d, b in rr.buffers[name].items():
                        bad, first = oracle_compare_device(w.model, p, self.c, d, seed, b.ptr, b.nbytes)
                        if bad:
                            self.failures.append(f"7B {name} shard {d}: {bad} mismatches (first byte {first})")
                if rr.relay_timeouts() or rr.barrier.timed_out():
                    self.failures.append("7B: flag or barrier timeouts")
                dist.barrier()
            finally:
                rr.close()

    def finish(self, sections) -> int:
        if self.world > 1 and "staged" in sections and self.staged_phases == 0:
            self.failures.append("staged cases ran no staged phase")
        t = torch.tensor([self.ce_runs], device="cpu" if self.oversub else "cuda")
        dist.all_reduce(t)
        if self.world > 1 and ("ce" in sections or "cetransport" in sections) and t.item() == 0:
            self.failures.append("copy-engine cases issued no runs")
        flag = torch.tensor([len(self.failures)], device="cpu" if self.oversub else "cuda")
        dist.all_reduce(flag)
        for f in self.failures:
            print(f"rank {self.rank}: {f}", flush=True)
        if self.rank == 0:
            print(f"dist_worker: copy-engine runs {t.item()} (all ranks), staged phases on rank 0: "
                  f"{self.staged_phases}", flush=True)
            print(f"dist_worker world={self.world}: {'OK' if flag.item() == 0 else 'FAILED'}", flush=True)
        dist.destroy_process_group()
        return 0 if flag.item() == 0 else 1


def main() -> int:
    w = Worker()
    sections = os.environ.get("RR_SECTIONS",
                              "basic,multicast,overlap,relay,ce,cetransport,probe,nccl,staged,fuzz,full7b").split(",")
    table = {"basic": w.basic, "multicast": w.multicast, "overlap": w.overlap, "relay": w.relay,
             "ce": w.ce_runs_cases, "cetransport": w.ce_transport, "probe": w.probe, "nccl": w.nccl_scheme,
             "staged": w.staged, "staged_many": w.staged_many_items, "fuzz": w.fuzz,
             "full7b": w.full_7b}
    for s in sections + (["staged_many"] if "staged" in sections else []):
        table[s]()
    return w.finish(sections)


if __name__ == "__main__":
    sys.exit(main())
