"""Device-side execution of a ReallocPlan on B200s (through librrealloc.so).

This is the B200 replacement of the upstream model worker's
"Redistributing Parameters" step: there, sources NCCL-
broadcast TP partitions to destinations; here every source GPU runs one
sm_100a kernel that gathers its slices and stores them straight into the
destination shards — locally through HBM, remotely through NVLink peer
stores — with no pack/unpack pass.

Two deployment shapes:

* ``VirtualCluster`` — all plan devices hosted on one CUDA device (the
  1-GPU local-relayout configuration and the single-GPU parity tests).
* ``RankRealloc`` — one process per GPU (torchrun), each hosting a
  contiguous block of plan devices; destination shards are exchanged as
  CUDA IPC handles through ``torch.distributed`` and a flag barrier over
  peer memory orders the phases.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import numpy as np

from ._lib import RrExecOptions, check, lib
from .rlplan import ReallocPlan

PUSH, PULL = 0, 1
SRC, DST = 0, 1
# Copy kernel unless a caller picks one (rr_exec_set_kernel): None keeps the
# library default, the TMA bulk ring (4 x 16 KiB stages, 3 CTAs per SM;
# profiles/r01_sweep_kernels.txt) with the LDG/STG kernel for plain phases
# storing < 64 MiB (profiles/r01_launch_latency_n1.json).
DEFAULT_KERNEL = None
# ... and for flag-synchronised phases (rr_exec_set_flag_kernel): 3 x 16 KiB
# stages, 4 CTAs per SM (profiles/r01_flag_kernel_sweep_n{2,4}.txt).
DEFAULT_FLAG_KERNEL = 5


def _stream_ptr(stream) -> Optional[int]:
    """Accept None, an int cudaStream_t, or a torch.cuda.Stream."""
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


def device_count() -> int:
    n = ctypes.c_int()
    check(lib.rr_device_count(ctypes.byref(n)))
    return n.value


class DeviceBuffer:
    """A cudaMalloc allocation owned by the library (IPC-exportable)."""

    def __init__(self, cuda_device: int, nbytes: int):
        self.cuda_device, self.nbytes = cuda_device, nbytes
        p = ctypes.c_void_p()
        check(lib.rr_device_alloc(cuda_device, max(nbytes, 256), ctypes.byref(p)))
        self.ptr: int = p.value

    def zero(self, stream=None) -> None:
        check(lib.rr_memset(self.ptr, 0, max(self.nbytes, 256), _stream_ptr(stream)))

    def ipc_handle(self) -> bytes:
        h = ctypes.create_string_buffer(64)
        check(lib.rr_ipc_handle(self.ptr, h))
        return h.raw

    def to_host(self) -> np.ndarray:
        out = np.empty(self.nbytes // 2, dtype=np.uint16)
        if self.nbytes:
            check(lib.rr_memcpy(out.ctypes.data, self.ptr, self.nbytes, 1, None, 1))
        return out

    def from_host(self, arr: np.ndarray) -> None:
        arr = np.ascontiguousarray(arr)
        assert arr.nbytes <= max(self.nbytes, 256)
        check(lib.rr_memcpy(self.ptr, arr.ctypes.data, arr.nbytes, 0, None, 1))

    def free(self) -> None:
        if self.ptr:
            lib.rr_device_free(self.ptr)
            self.ptr = 0


class HostBuffer:
    """Pinned host memory (for the end-to-end host->device leg)."""

    def __init__(self, nbytes: int):
        self.nbytes = nbytes
        p = ctypes.c_void_p()
        check(lib.rr_host_alloc(max(nbytes, 256), ctypes.byref(p)))
        self.ptr: int = p.value

    def array(self) -> np.ndarray:
        buf = (ctypes.c_uint16 * (self.nbytes // 2)).from_address(self.ptr)
        return np.ctypeslib.as_array(buf)

    def free(self) -> None:
        if self.ptr:
            lib.rr_host_free(self.ptr)
            self.ptr = 0


def memcpy_async(dst: int, src: int, nbytes: int, kind: int, stream=None) -> None:
    """kind 0 host->device, 1 device->host, 2 device->device."""
    check(lib.rr_memcpy(dst, src, nbytes, kind, _stream_ptr(stream), 0))


def stream_sync(stream=None) -> None:
    check(lib.rr_stream_sync(_stream_ptr(stream)))


def fill_shard(plan: ReallocPlan, side: int, device: int, ptr: int, seed: int, stream=None) -> None:
    check(lib.rr_fill_shard(plan.handle, side, device, ptr, seed, _stream_ptr(stream)))


def verify_shard(plan: ReallocPlan, side: int, device: int, ptr: int, seed: int,
                 stream=None) -> Tuple[int, int]:
    """(mismatching elements, first mismatching element index or -1)."""
    bad, first = ctypes.c_int64(), ctypes.c_int64()
    check(lib.rr_verify_shard(plan.handle, side, device, ptr, seed, _stream_ptr(stream),
                              ctypes.byref(bad), ctypes.byref(first)))
    return bad.value, first.value


def weight_value(seed: int, tensor: int, index: int) -> int:
    return lib.rr_weight_value(seed, tensor, index)


class Executor:
    """A plan bound to buffers on one CUDA device (rr_exec_create).

    ``host_of`` (plan device -> GPU) enables hierarchical delivery: a payload
    for several plan devices of one remote GPU crosses NVLink once (phase 0)
    and that GPU replicates it locally (phase 1, ``launch_fanout``)."""

    def __init__(self, plan: ReallocPlan, cuda_device: int, src_ptrs: Dict[int, int], dst_ptrs: Dict[int, int],
                 local: Iterable[int], mode: int = PUSH, chunk_bytes: int = 0,
                 host_of: Optional[Sequence[int]] = None, mc_ptrs: Optional[Dict[int, int]] = None,
                 relay_flags: Optional[Dict[int, int]] = None, relay_chain: bool = True,
                 overlap_fanout: bool = False, ce_min_run_bytes: int = 0, stage_chunk_bytes: int = 0,
                 n_hosts: int = 0, stage_remote: Optional[Dict[Tuple[int, int], int]] = None,
                 stage_flags: Optional[Dict[int, int]] = None, ce_transport: int = 0,
                 ce_flags: Optional[Dict[int, int]] = None):
        n = plan.cluster.device_count()
        self.plan = plan
        sp, dp = (ctypes.c_void_p * n)(), (ctypes.c_void_p * n)()
        for d, p in src_ptrs.items():
            sp[d] = p
        for d, p in dst_ptrs.items():
            dp[d] = p
        loc = list(local)
        arr = (ctypes.c_int32 * max(1, len(loc)))(*loc)
        hosts = (ctypes.c_int32 * n)(*host_of) if host_of is not None else None
        mcs = None
        if mc_ptrs:
            mcs = (ctypes.c_void_p * n)()
            for d, p in mc_ptrs.items():
                mcs[d] = p
        rfl = None
        if relay_flags:
            rfl = (ctypes.c_void_p * n)()
            for d, p in relay_flags.items():
                rfl[d] = p
        srem = sfl = None
        if stage_chunk_bytes:
            srem = (ctypes.c_void_p * (n * n_hosts))()
            for (d, h), p in (stage_remote or {}).items():
                srem[d * n_hosts + h] = p
            sfl = (ctypes.c_void_p * n_hosts)()
            for h, p in (stage_flags or {}).items():
                sfl[h] = p
        cfl = None
        if ce_flags:
            cfl = (ctypes.c_void_p * n_hosts)()
            for h, p in ce_flags.items():
                cfl[h] = p
        opt = RrExecOptions(mode, chunk_bytes, hosts, mcs, rfl, int(relay_chain), int(overlap_fanout),
                            ce_min_run_bytes, stage_chunk_bytes, n_hosts, srem, sfl, int(ce_transport), cfl)
        h = ctypes.c_void_p()
        check(lib.rr_exec_create_ex(plan.handle, cuda_device, n, sp, dp, len(loc), arr, ctypes.byref(opt),
                                    ctypes.byref(h)))
        self._h = h
        self.items, self.bytes_written, self.bytes_read = self.stats(0)
        self.fanout_items, self.fanout_written, self.fanout_read = self.stats(1)
        wi, wo = ctypes.c_int64(), ctypes.c_int64()
        check(lib.rr_exec_wire(h, ctypes.byref(wi), ctypes.byref(wo)))
        self.wire_in, self.wire_out = wi.value, wo.value

    def stats(self, phase: int) -> Tuple[int, int, int]:
        """(items, bytes stored, bytes read) of phase 0 (direct) or 1 (fan-out)."""
        it, w, r = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(lib.rr_exec_stats(self._h, phase, ctypes.byref(it), ctypes.byref(w), ctypes.byref(r)))
        return it.value, w.value, r.value

    def launch(self, stream=None, ctas: int = 0) -> None:
        check(lib.rr_exec_launch(self._h, _stream_ptr(stream), ctas))

    def launch_fanout(self, stream=None, ctas: int = 0) -> None:
        check(lib.rr_exec_launch_fanout(self._h, _stream_ptr(stream), ctas))

    def relay_timeouts(self) -> int:
        out = ctypes.c_int64()
        check(lib.rr_exec_relay_timeouts(self._h, ctypes.byref(out)))
        return out.value

    def kernel_count(self) -> Tuple[int, int]:
        """Kernels one launch() / launch_fanout() issues."""
        a, b = ctypes.c_int(), ctypes.c_int()
        check(lib.rr_exec_kernel_count(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def ce_runs(self) -> Tuple[int, int]:
        """(copy-engine submissions — runs or transport copies —, their bytes)
        that launch() issues beside the kernels."""
        n, b = ctypes.c_int(), ctypes.c_int64()
        check(lib.rr_exec_ce_runs(self._h, ctypes.byref(n), ctypes.byref(b)))
        return n.value, b.value

    def stage_pushes(self) -> Tuple[int, int]:
        """(staged-gather pieces, their bytes) that launch() pushes per call."""
        n, b = ctypes.c_int(), ctypes.c_int64()
        check(lib.rr_exec_stage_pushes(self._h, ctypes.byref(n), ctypes.byref(b)))
        return n.value, b.value

    def phase_kernels(self, phase: int = 0) -> Tuple[bool, int]:
        """(LDG/STG kernel runs, TMA bulk variant that runs or 0) for a phase."""
        a, b = ctypes.c_int(), ctypes.c_int()
        check(lib.rr_exec_phase_kernels(self._h, phase, ctypes.byref(a), ctypes.byref(b)))
        return bool(a.value), b.value

    def enable_onload(self, src_bytes: Dict[int, int], chunk_bytes: int = 256 << 20) -> None:
        """Prepare onload pipelining: the local source shards {device: bytes}
        are copied host->device in chunk_bytes pieces (in device order)."""
        devs = sorted(src_bytes)
        arr = (ctypes.c_int32 * max(1, len(devs)))(*devs)
        sizes = (ctypes.c_int64 * max(1, len(devs)))(*[src_bytes[d] for d in devs])
        check(lib.rr_exec_enable_onload(self._h, len(devs), arr, sizes, chunk_bytes))

    def launch_onload(self, host_ptrs: Dict[int, int], copy_stream, stream=None, ctas: int = 0) -> None:
        """Phase 0 with its sources onloaded from pinned host memory on
        ``copy_stream``; each copy segment starts as soon as its chunk lands."""
        n = self.plan.cluster.device_count()
        hp = (ctypes.c_void_p * n)()
        for d, p in host_ptrs.items():
            hp[d] = p
        check(lib.rr_exec_launch_onload(self._h, hp, _stream_ptr(copy_stream), _stream_ptr(stream), ctas))

    def launch_offload(self, src_bytes: Dict[int, int], host_ptrs: Dict[int, int], copy_stream,
                       stream=None) -> None:
        """Park the local source shards {device: bytes} in pinned host memory
        (device -> host on ``copy_stream``, after the work already on
        ``stream``). A launch() that follows on ``stream`` overlaps it; write
        the sources only after ``copy_stream`` has drained."""
        n = self.plan.cluster.device_count()
        devs = sorted(src_bytes)
        arr = (ctypes.c_int32 * max(1, len(devs)))(*devs)
        sizes = (ctypes.c_int64 * max(1, len(devs)))(*[src_bytes[d] for d in devs])
        hp = (ctypes.c_void_p * n)()
        for d, p in host_ptrs.items():
            hp[d] = p
        check(lib.rr_exec_launch_offload(self._h, len(devs), arr, sizes, hp, _stream_ptr(copy_stream),
                                         _stream_ptr(stream)))

    def set_kernel(self, kernel: int) -> None:
        """0 = LDG/STG kernel, 1 = TMA bulk ring (4 x 16 KiB stages), 5 = TMA bulk ring (3 x 16 KiB)."""
        check(lib.rr_exec_set_kernel(self._h, kernel))

    def set_flag_kernel(self, kernel: int) -> None:
        """The kernel of flag-synchronised phases (relay / overlapped fan-out)."""
        check(lib.rr_exec_set_flag_kernel(self._h, kernel))

    def close(self) -> None:
        if self._h and self._h.value:
            lib.rr_exec_destroy(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        self.close()


class VirtualCluster:
    """Every device of a plan hosted on one CUDA device.

    Allocates the source shards of the plan's source placement and the
    destination shards of its destination placement, each zeroed (padding
    bytes are therefore deterministic)."""

    def __init__(self, plan: ReallocPlan, cuda_device: int = 0):
        self.plan, self.cuda_device = plan, cuda_device
        self.src: Dict[int, DeviceBuffer] = {}
        self.dst: Dict[int, DeviceBuffer] = {}
        for d in plan.devices(SRC):
            self.src[d] = DeviceBuffer(cuda_device, plan.shard_bytes(SRC, d))
            self.src[d].zero()
        for d in plan.devices(DST):
            self.dst[d] = DeviceBuffer(cuda_device, plan.shard_bytes(DST, d))
            self.dst[d].zero()
        stream_sync()

    def fill_sources(self, seed: int) -> None:
        for d, b in self.src.items():
            fill_shard(self.plan, SRC, d, b.ptr, seed)

    def executor(self, mode: int = PUSH, chunk_bytes: int = 0, kernel: Optional[int] = DEFAULT_KERNEL) -> Executor:
        devs = sorted(set(self.src) | set(self.dst))
        ex = Executor(self.plan, self.cuda_device, {d: b.ptr for d, b in self.src.items()},
                      {d: b.ptr for d, b in self.dst.items()}, devs, mode, chunk_bytes)
        if kernel is not None:
            ex.set_kernel(kernel)
        return ex

    def verify_destinations(self, seed: int) -> Dict[int, Tuple[int, int]]:
        return {d: verify_shard(self.plan, DST, d, b.ptr, seed) for d, b in self.dst.items()}

    def free(self) -> None:
        for b in list(self.src.values()) + list(self.dst.values()):
            b.free()


class Barrier:
    """Cross-GPU barrier for one-process-per-GPU runs (rr_barrier_*).

    Each rank owns a `world`-entry uint32 flag array; rank r's launch stores
    the epoch into every peer's slot r (st.release.sys) and waits until all
    its own slots reach the epoch (ld.acquire.sys, bounded spin)."""

    def __init__(self, cuda_device: int, rank: int, world: int, flag_ptrs: Sequence[int]):
        arr = (ctypes.c_void_p * world)(*flag_ptrs)
        h = ctypes.c_void_p()
        check(lib.rr_barrier_create(cuda_device, rank, world, arr, ctypes.byref(h)))
        self._h = h

    def launch(self, stream=None) -> None:
        check(lib.rr_barrier_launch(self._h, _stream_ptr(stream)))

    def timed_out(self) -> bool:
        out = ctypes.c_int()
        check(lib.rr_barrier_status(self._h, ctypes.byref(out)))
        return bool(out.value)

    def close(self) -> None:
        if self._h and self._h.value:
            lib.rr_barrier_destroy(self._h)
            self._h = ctypes.c_void_p(0)


def open_ipc(cuda_device: int, handle: bytes) -> int:
    p = ctypes.c_void_p()
    check(lib.rr_ipc_open(cuda_device, handle, ctypes.byref(p)))
    return p.value


def close_ipc(ptr: int) -> None:
    lib.rr_ipc_close(ptr)


def hosted_devices(n_plan_devices: int, rank: int, world: int) -> List[int]:
    """Contiguous block of plan devices hosted by `rank` (world | n)."""
    if n_plan_devices % world:
        raise ValueError(f"{world} ranks cannot evenly host {n_plan_devices} plan devices")
    k = n_plan_devices // world
    return list(range(rank * k, (rank + 1) * k))


def _all_gather_shaped(plan: ReallocPlan, host_of: Sequence[int], world: int, ce_min_run_bytes: int = 0) -> bool:
    """Every GPU both sends sources to and receives sources from others,
    every GPU that reads a remote source shard reads (>= 98% of) all of it
    (the staged gather moves whole shards), each GPU receives >= 1 GiB, and
    no range moves as a copy-engine run already (stage remaps)."""
    needs = [False] * world
    sends = [False] * world
    read: Dict[Tuple[int, int], int] = {}
    for s, dsts, rects in plan.lowered():
        b = sum(r[2] * r[5] for r in rects)
        for h in {host_of[d] for d in dsts if host_of[d] != host_of[s]}:
            needs[h] = True
            sends[host_of[s]] = True
            read[(s, h)] = read.get((s, h), 0) + b
    if not (all(needs) and all(sends)):
        return False
    if any(b * 50 < plan.shard_bytes(SRC, s) * 49 for (s, _h), b in read.items()):
        return False
    # small phases stay on SM stores: copy-engine submissions and piece
    # signals cost microseconds each
    received = [0] * world
    for (s, h), b in read.items():
        received[h] += b
    if min(received) < (1 << 30):
        return False
    if ce_min_run_bytes < 0:  # copy-engine runs switched off: none to defer to
        return True
    n = plan.cluster.device_count()
    min_run = ce_min_run_bytes or (256 << 20)  # 0 = the library default
    return not any(plan.ce_runs([d for d in range(n) if host_of[d] == r], host_of, min_run) for r in range(world))


# Measured NVLink rates (profiles/r01_nvlink_probe_n2.txt, r01_ce_probe_*):
# SM peer stores cap at ~705 GB/s of payload per GPU, a copy engine moves
# ~775 GB/s pairwise and costs ~4 us per submission.
SM_LINK_GBS, CE_LINK_GBS, CE_COPY_S = 705e9, 775e9, 4e-6


HBM_COPY_GBS = 6.5e12  # measured 1:1 device copy (MEASURED_PEAKS.json)
PHASE_OVERHEAD_S = 30e-6  # a barrier + fan-out launch


def fanout_bytes(plan: ReallocPlan, host_of: Sequence[int]) -> Dict[int, int]:
    """Per host: bytes its in-host fan-out copies from leader replicas (a
    payload reaching k >= 2 destinations on a remote host crosses once and is
    replicated k - 1 times there)."""
    out = {h: 0 for h in set(host_of)}
    for s, dsts, rects in plan.lowered():
        b = sum(r[2] * r[5] for r in rects)
        per: Dict[int, int] = {}
        for d in dsts:
            if host_of[d] != host_of[s]:
                per[host_of[d]] = per.get(host_of[d], 0) + 1
        for h, k in per.items():
            out[h] += (k - 1) * b
    return out


def ce_transport_estimate(plan: ReallocPlan, host_of: Sequence[int], star: bool = False) -> Tuple[float, float]:
    """Predicted time (s) of a phase: (copy-engine transport, SM peer stores
    with the in-host fan-out overlapped), each the max over hosts of link
    time (sending and receiving at the measured rates) and HBM time (host
    only). Without `star` the copy-engine side runs the in-host fan-out as a
    separate phase after it; with it (copy-engine star) the fan-out overlaps."""
    n = plan.cluster.device_count()
    hosts = sorted(set(host_of))
    recv = {h: 0 for h in hosts}
    ce_send = {h: 0.0 for h in hosts}
    hbm = {h: 0.0 for h in hosts}
    sm = 0.0
    for h in hosts:
        local = [d for d in range(n) if host_of[d] == h]
        copies = plan.ce_copies(local, host_of)
        for c in copies:
            recv[host_of[c[1]]] += c[4] * c[5] * c[6]
        ce_send[h] = sum(c[4] * c[5] * c[6] for c in copies) / CE_LINK_GBS + len(copies) * CE_COPY_S
        w = plan.work(local, PUSH, host_of)
        # bytes this GPU's HBM reads and writes: local reads, stores landing
        # here (local and incoming), the fan-out's reads and writes
        hbm[h] = (w["read"] + w["written"] - w["wire_out"] + w["wire_in"] + w["fanout_read"] +
                  w["fanout_written"]) / HBM_COPY_GBS
        sm = max(sm, max(w["wire_in"], w["wire_out"]) / SM_LINK_GBS, hbm[h])
    fan = fanout_bytes(plan, host_of)
    # the copy engines follow the library's schedule (receiver chains): its
    # simulated makespan, not just each host's bytes, bounds the link time
    sched = plan.ce_schedule(host_of)
    makespan = max((t[3] for t in sched), default=0.0)
    ce = max(max(ce_send[h], recv[h] / CE_LINK_GBS, hbm[h], makespan) for h in hosts)
    if any(fan.values()) and not star:
        ce += max(2 * fan[h] for h in hosts) / HBM_COPY_GBS + PHASE_OVERHEAD_S
    return ce, sm


def ce_slots(plan: ReallocPlan, host_of: Sequence[int]) -> int:
    """Length of the copy flag array every host allocates (copy-engine star)."""
    n = plan.cluster.device_count()
    hosts = (ctypes.c_int32 * n)(*host_of)
    out = ctypes.c_int64()
    check(lib.rr_plan_ce_slots(plan.handle, hosts, ctypes.byref(out)))
    return out.value


def stage_slots(plan: ReallocPlan, host_of: Sequence[int], chunk_bytes: int) -> int:
    """Length of the stage flag array every host allocates for a staged gather."""
    n = plan.cluster.device_count()
    hosts = (ctypes.c_int32 * n)(*host_of)
    out = ctypes.c_int64()
    check(lib.rr_plan_stage_slots(plan.handle, hosts, chunk_bytes, ctypes.byref(out)))
    return out.value


def relay_slots(plan: ReallocPlan, host_of: Sequence[int], chunk_bytes: int = 0, chain: bool = True,
                overlap: bool = False) -> int:
    """Length of the relay flag array for this host map and scheme switches
    (same on every rank)."""
    n = plan.cluster.device_count()
    hosts = (ctypes.c_int32 * n)(*host_of)
    out = ctypes.c_int64()
    check(lib.rr_plan_relay_slots(plan.handle, hosts, chunk_bytes, int(chain), int(overlap), ctypes.byref(out)))
    return out.value


def link_bottleneck(plan: ReallocPlan, host_of: Sequence[int], multicast: bool = False, relay: bool = False) -> int:
    """Estimated bottleneck link bytes of a GPU (max over hosts of max(egress,
    ingress)) for hierarchical push delivery, optionally with NVLS multicast
    of payloads that reach every host (the switch also loops the source's own
    copy back, so multicast adds ingress at the source) or with the pipelined
    relay for payloads reaching >= 2 other hosts (every chain host receives
    one copy, all but the last send one)."""
    hosts = set(host_of)
    egress = {h: 0 for h in hosts}
    ingress = {h: 0 for h in hosts}
    for s, dsts, rects in plan.lowered():
        b = sum(r[2] * r[5] for r in rects)
        hs = host_of[s]
        dst_hosts = {host_of[d] for d in dsts}
        remote = dst_hosts - {hs}
        if relay and len(remote) >= 2:
            chain = sorted(remote, key=lambda h: (h - hs) % (max(hosts) + 1))
            egress[hs] += b
            for k, h in enumerate(chain):
                ingress[h] += b
                if k + 1 < len(chain):
                    egress[h] += b
        elif multicast and dst_hosts == hosts and remote:
            egress[hs] += b
            for h in dst_hosts:
                ingress[h] += b
        else:
            egress[hs] += b * len(remote)
            for h in remote:
                ingress[h] += b
    return max(max(egress[h], ingress[h]) for h in hosts)


def multicast_supported(cuda_device: int = 0) -> bool:
    out = ctypes.c_int()
    check(lib.rr_mcast_supported(cuda_device, ctypes.byref(out)))
    return bool(out.value)


_MC_COUNTER = [0]


def _share_fd(fd: int, rank: int, world: int, tag: str, group=None) -> int:
    """Pass rank 0's file descriptor to every rank (SCM_RIGHTS over an
    abstract AF_UNIX socket; all ranks are on one host)."""
    import socket

    import torch.distributed as dist
    name = "\0" + tag
    if rank == 0:
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(name)
        srv.listen(world)
        dist.barrier(group=group)
        for _ in range(world - 1):
            conn, _ = srv.accept()
            socket.send_fds(conn, [b"fd"], [fd])
            conn.close()
        srv.close()
        dist.barrier(group=group)
        return fd
    dist.barrier(group=group)
    s = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    s.connect(name)
    _msg, fds, _flags, _addr = socket.recv_fds(s, 16, 1)
    s.close()
    dist.barrier(group=group)
    return fds[0]


def _exchange_fds(fd: int, rank: int, world: int, tag: str, group=None) -> List[int]:
    """Every rank's file descriptor to every rank (rank r serves its fd on an
    abstract AF_UNIX socket in turn r; SCM_RIGHTS). Entry `rank` is `fd`."""
    import socket

    import torch.distributed as dist
    out = [-1] * world
    out[rank] = fd
    for r in range(world):
        name = "\0" + f"{tag}-{r}"
        if rank == r:
            srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            srv.bind(name)
            srv.listen(world)
            dist.barrier(group=group)
            for _ in range(world - 1):
                conn, _ = srv.accept()
                socket.send_fds(conn, [b"fd"], [fd])
                conn.close()
            srv.close()
        else:
            dist.barrier(group=group)
            c = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            c.connect(name)
            _msg, fds, _flags, _addr = socket.recv_fds(c, 16, 1)
            c.close()
            out[r] = fds[0]
        dist.barrier(group=group)
    return out


class PeerMemory:
    """Another GPU's multicast member mapped here for ordinary peer stores
    (rr_peer_mem_import)."""

    def __init__(self, cuda_device: int, fd: int, nbytes: int):
        p, h = ctypes.c_void_p(), ctypes.c_void_p()
        check(lib.rr_peer_mem_import(cuda_device, fd, nbytes, ctypes.byref(p), ctypes.byref(h)))
        self.ptr, self._h = p.value, h

    def close(self) -> None:
        if self._h and self._h.value:
            lib.rr_peer_mem_close(self._h)
            self._h = ctypes.c_void_p(0)


class MulticastBuffer:
    """One rank's member buffer of an NVLS multicast object (rr_mcast_*).

    Collective over the process group: rank 0 creates the object, the others
    import it through its file descriptor, every rank adds its GPU, then
    (after a barrier) binds local memory. ``ptr`` is the ordinary (unicast)
    address of this rank's member; ``mc_ptr`` the multicast address through
    which one store reaches every member."""

    def __init__(self, cuda_device: int, nbytes: int, rank: int, world: int, group=None):
        import os

        import torch.distributed as dist
        self.cuda_device, self.nbytes = cuda_device, nbytes
        h = ctypes.c_void_p()
        meta = [None]
        if rank == 0:
            fd, size = ctypes.c_int(), ctypes.c_size_t()
            check(lib.rr_mcast_create(cuda_device, max(nbytes, 256), world, ctypes.byref(fd), ctypes.byref(size),
                                      ctypes.byref(h)))
            _MC_COUNTER[0] += 1
            meta = [(fd.value, size.value, f"rr-mcast-{os.getpid()}-{_MC_COUNTER[0]}")]
        dist.broadcast_object_list(meta, src=0, group=group)
        fd0, size, tag = meta[0]
        fd_local = _share_fd(fd0 if rank == 0 else -1, rank, world, tag, group)
        if rank != 0:
            check(lib.rr_mcast_import(cuda_device, fd_local, size, world, ctypes.byref(h)))
            os.close(fd_local)
        self._h = h
        dist.barrier(group=group)  # every GPU added before anyone binds memory
        uc, mc = ctypes.c_void_p(), ctypes.c_void_p()
        check(lib.rr_mcast_bind(h, ctypes.byref(uc), ctypes.byref(mc)))
        dist.barrier(group=group)
        self.ptr, self.mc_ptr, self.padded = uc.value, mc.value, size

    def zero(self, stream=None) -> None:
        check(lib.rr_memset(self.ptr, 0, self.padded, _stream_ptr(stream)))

    def to_host(self) -> np.ndarray:
        out = np.empty(self.nbytes // 2, dtype=np.uint16)
        if self.nbytes:
            check(lib.rr_memcpy(out.ctypes.data, self.ptr, self.nbytes, 1, None, 1))
        return out

    def export_fd(self) -> int:
        """This member's physical memory as a POSIX fd (peers map it with
        PeerMemory for ordinary peer stores)."""
        fd = ctypes.c_int()
        check(lib.rr_mcast_export_member(self._h, ctypes.byref(fd)))
        return fd.value

    def free(self) -> None:
        if self._h and self._h.value:
            lib.rr_mcast_destroy(self._h)
            self._h = ctypes.c_void_p(0)
            self.ptr = 0


@dataclass(frozen=True)
class Scheme:
    """How one phase's remote pieces travel (RankRealloc). All are bit-exact;
    they differ in which engine carries the bytes and when in-host fan-outs
    run."""
    relay: bool = False         # pipelined relay chain for payloads reaching >= 2 other GPUs
    overlap: bool = False       # per-chunk in-host fan-out inside phase 0 (star flags)
    staged: bool = False        # copy-engine rotation of whole shards + per-piece unpack
    ce_transport: bool = False  # copy-engine 2D/3D copies straight into the destinations
    ce_hybrid: bool = False     # ... with unmerged row-parallel pieces left on SM peer stores
    nccl: bool = False          # the library baseline: NCCL moves whole source shards, then a local unpack
    multicast: bool = False     # NVLS multicast: a payload for every GPU stored once through multimem.st

    def label(self) -> str:
        parts = [k for k in ("relay", "overlap", "staged", "ce_transport", "ce_hybrid", "nccl", "multicast")
                 if getattr(self, k)]
        return "+".join(parts) or "push"


def _torch_bytes(ptr: int, nbytes: int):
    """A torch uint8 tensor aliasing device memory the library allocated."""
    import torch

    class _View:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}
    return torch.as_tensor(_View(), device="cuda")


class NcclStaged:
    """The NCCL baseline as a delivery scheme (the upstream runtime moves
    weights with NCCL): every source shard another rank reads
    moves whole with NCCL — `broadcast` when one source shard feeds every
    rank, else `batch_isend_irecv` to exactly the ranks that read it — into
    staging buffers, then the library's pull executor unpacks it locally.
    Behaves like an Executor (launch, stats, onload) so that the bind-time
    probe times it beside the library's own schemes on the same buffers."""

    def __init__(self, inner: "Executor", group, sends, recvs, bcast, local_src: Dict[int, "DeviceBuffer"]):
        self.inner, self.group = inner, group
        self.sends, self.recvs, self.bcast = sends, recvs, bcast  # lists of (tensor, peer rank)
        self.local_src = local_src
        self._onload = None

    def __getattr__(self, name):  # stats, wire, kernel_count, phase_kernels, ... of the unpack executor
        return getattr(self.inner, name)

    def _collective(self) -> None:
        import torch.distributed as dist
        if self.bcast is not None:
            t, root = self.bcast
            dist.broadcast(t, src=root, group=self.group)
            return
        ops = [dist.P2POp(dist.isend, t, q, group=self.group) for t, q in self.sends]
        ops += [dist.P2POp(dist.irecv, t, q, group=self.group) for t, q in self.recvs]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def launch(self, stream=None, ctas: int = 0) -> None:
        self._collective()  # ordered after the work on torch's current stream
        self.inner.launch(stream, ctas)

    def enable_onload(self, src_bytes: Dict[int, int], chunk_bytes: int = 256 << 20) -> None:
        self._onload = dict(src_bytes)

    def launch_onload(self, host_ptrs: Dict[int, int], copy_stream, stream=None, ctas: int = 0) -> None:
        # the baseline is not pipelined: the local sources land, then NCCL, then the unpack
        for d, nb in (self._onload or {}).items():
            memcpy_async(self.local_src[d].ptr, host_ptrs[d], nb, 0, stream)
        self.launch(stream, ctas)

    def ce_runs(self) -> Tuple[int, int]:
        return 0, 0

    def stage_pushes(self) -> Tuple[int, int]:
        return 0, 0

    def close(self) -> None:
        self.inner.close()


class _Binding:
    """One phase bound to a scheme: its executor and the flag / staging
    buffers it needs (allocated here, exchanged through CUDA IPC)."""

    def __init__(self):
        self.executor: Optional[Executor] = None
        self.owned: List[DeviceBuffer] = []
        self.opened: List[int] = []

    def free(self) -> None:
        if self.executor is not None:
            self.executor.close()
        for p in self.opened:
            close_ipc(p)
        for b in self.owned:
            b.free()
        self.executor, self.opened, self.owned = None, [], []


class RankRealloc:
    """One rank of a one-process-per-GPU reallocation.

    ``plans`` is a sequence of phases (e.g. train->gen, then gen->train); all
    use the same cluster devices. Each phase gets its own executor; phase i's
    destination shards must be phase i+1's source shards when chained, which
    the caller expresses through ``shards``: a dict name -> (plan index, side)
    telling which buffers to allocate, and ``bind``: per phase the (src name,
    dst name). Buffers of remote hosts are mapped through CUDA IPC; a barrier
    runs after every phase so the next phase reads completed shards.

    Per phase a delivery scheme (Scheme) is chosen: from the switches and the
    measured-rate cost model, or — with ``probe=True`` — by timing every
    scheme the switches allow on the real buffers at bind time (max over
    ranks, a few launches each) and keeping the fastest (``probe_log``).
    """

    def __init__(self, plans: Sequence[ReallocPlan], shards: Dict[str, Tuple[int, int]],
                 bind: Sequence[Tuple[str, str]], rank: int, world: int, cuda_device: int, group=None,
                 mode: int = PUSH, kernel: Optional[int] = DEFAULT_KERNEL, hierarchical: bool = True,
                 multicast: Sequence[str] = (), relay=False, overlap: bool = False,
                 flag_kernel: int = DEFAULT_FLAG_KERNEL, chunk_bytes: int = 0, ce_min_run_bytes: int = 0,
                 staged=False, stage_chunk_bytes: int = 512 << 20, ce_transport=False, probe: bool = False):
        """``multicast`` names shard sets whose per-GPU leader shards (the
        lowest-id plan device of the set on each GPU) are members of one NVLS
        multicast object: a payload bound for every GPU is then stored once
        (K3) instead of once per GPU (needs world > 1, push mode,
        hierarchical delivery). ``chunk_bytes``: work-item size (0 = the
        library default), also the relay/overlap flag granularity.
        ``relay`` / ``staged`` / ``ce_transport``: False, True (every phase
        it applies to) or "auto" (cost model); ``overlap``: bool."""
        self.plans, self.rank, self.world, self.cuda_device = list(plans), rank, world, cuda_device
        self.group, self.mode, self.kernel, self.flag_kernel = group, mode, kernel, flag_kernel
        self.hierarchical, self.chunk_bytes, self.ce_min_run_bytes = hierarchical, chunk_bytes, ce_min_run_bytes
        self.stage_chunk = stage_chunk_bytes
        n = plans[0].cluster.device_count()
        self.n = n
        self.local = hosted_devices(n, rank, world)
        self.owner = {d: d // (n // world) for d in range(n)}
        self.host_of = [self.owner[d] for d in range(n)]
        self.bind = list(bind)
        # Multicast sets: destination sets whose per-GPU leaders are members of
        # an NVLS multicast object. A list: those sets, multicast always.
        # "auto": with the probe, every set some payload of which reaches
        # every GPU, multicast kept only where the probe measures it fastest
        # (the members are also mapped by the peers for the other schemes);
        # without it, none. The link-byte model favours multicast wherever one
        # source feeds many GPUs, but multicast stores measured slower than
        # peer stores on every config (7B 28.0 vs 13.0 ms at
        # 2 GPUs), so only a measurement may choose it.
        self.mc_forced = multicast != "auto"
        if multicast == "auto":
            multicast = []
            # (one member per GPU: ranks sharing a GPU, as in the 8-ranks-on-4
            # correctness runs, cannot form a multicast group)
            if (probe and world > 1 and mode == PUSH and hierarchical and world <= device_count() and
                    multicast_supported(cuda_device)):
                for pi, (_sname, dname) in enumerate(bind):
                    p = self.plans[pi]
                    every = any({self.host_of[d] for d in dsts} == set(self.host_of) and
                                any(self.host_of[d] != self.host_of[s_] for d in dsts)
                                for s_, dsts, _r in p.lowered())
                    if every and dname not in multicast:
                        multicast.append(dname)
        self.multicast = list(multicast)
        if multicast and (world < 2 or mode != PUSH or not hierarchical):
            raise ValueError("multicast needs world > 1, push mode and hierarchical delivery")
        self.ce_estimates: Dict[int, Tuple[float, float]] = {}
        switches = dict(relay=relay, overlap=overlap, staged=staged, ce_transport=ce_transport)
        self.schemes: List[Scheme] = [self._decide(pi, switches) for pi in range(len(self.plans))]
        self._alloc_shards(shards)
        self.bindings: List[Optional[_Binding]] = [None] * len(self.plans)
        self.executors: List[Executor] = []
        self.has_fanout: List[bool] = [False] * len(self.plans)
        self.probe_log: List[dict] = []
        for pi in range(len(self.plans)):
            cands = self._candidates(pi, switches) if probe else [self.schemes[pi]]
            if len(cands) > 1:
                self.schemes[pi] = self._probe(pi, cands)
            self._bind_phase(pi, self.schemes[pi])
        self.executors = [b.executor for b in self.bindings]

    # ---- scheme choice ----------------------------------------------------

    def _flag_ok(self) -> bool:
        return self.world > 1 and self.mode == PUSH and self.hierarchical

    def _remote(self, p: ReallocPlan) -> bool:
        return any(self.host_of[s] != self.host_of[d] for s, dsts, _r in p.lowered() for d in dsts)

    def _decide(self, pi: int, sw: dict) -> Scheme:
        """The cost-model choice for phase pi under the switches."""
        p, dname = self.plans[pi], self.bind[pi][1]
        if dname in self.multicast and self.mc_forced and self._remote(p):
            return Scheme(multicast=True)
        if not self._flag_ok() or not self._remote(p):
            return Scheme()
        relay = bool(sw["relay"]) and (sw["relay"] != "auto" or link_bottleneck(p, self.host_of, relay=True) <
                                       0.9 * link_bottleneck(p, self.host_of))
        if relay:
            # ce_transport=True: the relay chains run on copy engines
            return Scheme(relay=True, overlap=bool(sw["overlap"]), ce_transport=sw["ce_transport"] is True)
        # Staged gather: True = every phase with remote reads; "auto" = from 4
        # GPUs on, all-gather-shaped phases that copy-engine runs do not cover.
        if sw["staged"] and (sw["staged"] != "auto" or (
                self.world >= 4 and _all_gather_shaped(p, self.host_of, self.world, self.ce_min_run_bytes))):
            return Scheme(staged=True)
        # Copy-engine transport: True = every remaining phase with remote
        # traffic; "auto" = where the measured rates predict >= 5% less time
        # than SM peer stores (ce_transport_estimate charges the copy-engine
        # side a separate in-host fan-out phase).
        # With overlap, the fan-out rides on per-copy flags (copy-engine star).
        if sw["ce_transport"]:
            star = bool(sw["overlap"]) and any(fanout_bytes(p, self.host_of).values())
            if sw["ce_transport"] != "auto":
                return Scheme(overlap=star, ce_transport=True)
            est = self.ce_estimates[pi] = ce_transport_estimate(p, self.host_of, star)
            if est[0] < 0.95 * est[1]:
                return Scheme(overlap=star, ce_transport=True)
        return Scheme(overlap=bool(sw["overlap"]))

    def _candidates(self, pi: int, sw: dict) -> List[Scheme]:
        """Every scheme the switches allow for phase pi (probe mode)."""
        p, dname = self.plans[pi], self.bind[pi][1]
        if dname in self.multicast and self.mc_forced:
            return [self.schemes[pi]]
        if not self._flag_ok() or not self._remote(p):
            return [Scheme()]
        out = [self.schemes[pi], Scheme(overlap=bool(sw["overlap"]))]
        if dname in self.multicast:
            out.append(Scheme(multicast=True))
        if sw["relay"] and any(len({self.host_of[d] for d in dsts} - {self.host_of[s]}) >= 2
                               for s, dsts, _r in p.lowered()):
            out.append(Scheme(relay=True, overlap=bool(sw["overlap"])))
            if sw["ce_transport"]:  # relay chains on copy engines
                out.append(Scheme(relay=True, overlap=bool(sw["overlap"]), ce_transport=True))
        if sw["staged"]:
            out.append(Scheme(staged=True))
        if self._nccl_ok():
            out.append(Scheme(nccl=True))  # the library baseline, timed beside the rest
        if sw["ce_transport"]:
            out.append(Scheme(ce_transport=True))
            if sw["overlap"] and any(fanout_bytes(p, self.host_of).values()):
                out.append(Scheme(overlap=True, ce_transport=True))
            # row-parallel pieces that stay per-layer 2D copies (thousands of
            # rows, depth 1): try them on SM stores beside the copy engines
            # (every host's copies: all ranks must build the same list)
            if any(c[6] == 1 and c[5] > 256 for r in range(self.world)
                   for c in p.ce_copies([d for d in range(self.n) if self.host_of[d] == r], self.host_of)):
                out.append(Scheme(ce_transport=True, ce_hybrid=True))
        uniq: List[Scheme] = []
        for sc in out:
            if sc not in uniq and self._fits(pi, sc):
                uniq.append(sc)
        return uniq or [self.schemes[pi]]

    def _nccl_ok(self) -> bool:
        if self.world < 2:
            return False
        import torch.distributed as dist
        return dist.get_backend(self.group) == "nccl"

    def _remote_sources(self, pi: int) -> List[int]:
        """Source devices on other ranks whose bytes this rank reads."""
        p = self.plans[pi]
        return sorted({s for s, dsts, _r in p.lowered() if self.host_of[s] != self.rank and
                       any(self.host_of[d] == self.rank for d in dsts)})

    def _fits(self, pi: int, sc: Scheme) -> bool:
        """Whether every rank has the device memory the scheme's extra buffers
        need (the staged gather stages whole remote source shards; 70B at 2
        GPUs would need 70 GB more than the 180 GB). Collective: all ranks
        agree."""
        need = 0
        if sc.staged or sc.nccl:
            p = self.plans[pi]
            need = sum(p.shard_bytes(SRC, s) for s in self._remote_sources(pi))
            if sc.nccl:  # a broadcast receives into a scratch buffer where nothing is read
                need += max(p.shard_bytes(SRC, s) for s in p.devices(SRC))
        ok = True
        if need:
            import torch
            ok = need < 0.9 * torch.cuda.mem_get_info(self.cuda_device)[0]
        return all(self._exchange({"ok": ok})[r]["ok"] for r in range(self.world)) if self.world > 1 else ok

    def _probe(self, pi: int, cands: List[Scheme], reps: int = 3) -> Scheme:
        """Bind each candidate, time `reps` launches of phase pi (after one
        warm-up) with CUDA events, take the max over ranks of the median, keep
        the fastest. Phase pi's destinations are overwritten (bind time: the
        caller fills sources afterwards)."""
        import torch
        timings: Dict[str, float] = {}
        best, best_ms = cands[0], float("inf")
        stream = torch.cuda.current_stream()
        for sc in cands:
            self._bind_phase(pi, sc)
            ex = self.bindings[pi].executor
            ms = []
            for k in range(reps + 1):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                self._collective_barrier()
                e0.record(stream)
                ex.launch(stream)
                self._finish_phase(pi, stream, 0)
                e1.record(stream)
                torch.cuda.synchronize()
                if k:
                    ms.append(e0.elapsed_time(e1))
            med = sorted(ms)[len(ms) // 2]
            med = self._allreduce_max(med)
            timings[sc.label()] = round(med, 4)
            if med < best_ms:
                best, best_ms = sc, med
            self._unbind_phase(pi)
        self.probe_log.append({"phase": pi, "ms": timings, "chosen": best.label(),
                               "cost_model": self.schemes[pi].label()})
        return best

    def _collective_barrier(self) -> None:
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier(group=self.group)

    def _allreduce_max(self, v: float) -> float:
        if self.world == 1:
            return v
        import torch.distributed as dist
        out: List[float] = [None] * self.world  # type: ignore
        dist.all_gather_object(out, v, group=self.group)
        return max(out)

    def _exchange(self, mine: dict) -> List[dict]:
        """all_gather of small picklable tables (IPC handles)."""
        if self.world == 1:
            return [mine]
        import torch.distributed as dist
        out: List[dict] = [None] * self.world  # type: ignore
        dist.all_gather_object(out, mine, group=self.group)
        return out

    # ---- buffers and bindings -----------------------------------------------

    def _alloc_shards(self, shards: Dict[str, Tuple[int, int]]) -> None:
        """Shard buffers of every set (multicast members for multicast sets),
        the barrier flags, and the IPC exchange that maps every remote shard
        and flag array here."""
        n, rank, world = self.n, self.rank, self.world
        self.buffers: Dict[str, Dict[int, object]] = {}
        self.mc_tables: Dict[str, Dict[int, int]] = {}
        mc_leaders: Dict[str, int] = {}
        for name, (pi, side) in shards.items():
            p = self.plans[pi]
            bufs = {}
            mine = [d for d in p.devices(side) if d in self.local]
            if name in self.multicast:
                if not mine:
                    raise ValueError(f"multicast set {name!r}: rank {rank} hosts none of its devices")
                import torch.distributed as dist
                leader = min(mine)
                sizes: List[int] = [None] * world  # type: ignore
                dist.all_gather_object(sizes, p.shard_bytes(side, leader), group=self.group)
                if len(set(sizes)) != 1:
                    raise ValueError(f"multicast set {name!r}: leader shards differ in size {sizes}")
                bufs[leader] = MulticastBuffer(self.cuda_device, sizes[0], rank, world, self.group)
                bufs[leader].zero()
                mc_leaders[name] = leader
                leaders = [min(d for d in p.devices(side) if d in hosted_devices(n, r, world)) for r in range(world)]
                self.mc_tables[name] = {d: bufs[leader].mc_ptr for d in leaders}
            for d in mine:
                if d in bufs:
                    continue
                bufs[d] = DeviceBuffer(self.cuda_device, p.shard_bytes(side, d))
                bufs[d].zero()
            self.buffers[name] = bufs
        self.flags = DeviceBuffer(self.cuda_device, 4 * max(world, 64))
        self.flags.zero()
        stream_sync()
        # multicast members are VMM allocations: reached through the multicast
        # address, not through CUDA IPC
        mine_h: dict = {}
        if world > 1:
            mine_h = {name: {d: b.ipc_handle() for d, b in bufs.items() if mc_leaders.get(name) != d}
                      for name, bufs in self.buffers.items()}
            mine_h["__flags__"] = {rank: self.flags.ipc_handle()}
        gathered = self._exchange(mine_h)
        self.ptrs: Dict[str, Dict[int, int]] = {name: {d: b.ptr for d, b in bufs.items()}
                                                 for name, bufs in self.buffers.items()}
        self._opened: List[int] = []
        flag_ptrs = [0] * world
        flag_ptrs[rank] = self.flags.ptr
        for r, table in enumerate(gathered):
            if r == rank:
                continue
            for name, handles in table.items():
                for d, h in handles.items():
                    ptr = open_ipc(self.cuda_device, h)
                    self._opened.append(ptr)
                    if name == "__flags__":
                        flag_ptrs[r] = ptr
                    else:
                        self.ptrs[name][d] = ptr
        self.barrier = Barrier(self.cuda_device, rank, world, flag_ptrs)
        # multicast members: every peer maps every other GPU's member for the
        # schemes that store with ordinary peer stores
        import os
        self._peer_mem: List[PeerMemory] = []
        for name, leader in sorted(mc_leaders.items()):
            b = self.buffers[name][leader]
            fd = b.export_fd()
            fds = _exchange_fds(fd, rank, world, f"rr-mem-{self._mc_tag()}-{name}", self.group)
            for r in range(world):
                if r == rank:
                    continue
                pm = PeerMemory(self.cuda_device, fds[r], b.padded)
                self._peer_mem.append(pm)
                peer_leader = min(d for d in self.plans[shards[name][0]].devices(shards[name][1])
                                  if d in hosted_devices(n, r, world))
                self.ptrs[name][peer_leader] = pm.ptr
                os.close(fds[r])
            os.close(fd)

    def _mc_tag(self) -> str:
        """A name every rank agrees on for this instance's fd sockets."""
        import os
        if not hasattr(self, "_tag"):
            tag = [f"{os.getpid()}-{id(self)}"]
            if self.world > 1:
                import torch.distributed as dist
                dist.broadcast_object_list(tag, src=0, group=self.group)
            self._tag = tag[0]
        return self._tag

    def _bind_phase(self, pi: int, sc: Scheme) -> None:
        """Allocate what scheme `sc` needs for phase pi (relay / overlap flag
        array, staging buffers and their flags), exchange it through IPC
        (collective), create the executor and agree on the fan-out step."""
        b = _Binding()
        rank, world, n = self.rank, self.world, self.n
        p = self.plans[pi]
        sname, dname = self.bind[pi]
        mine: dict = {}
        relay_buf = stage_flag = ce_flag = None
        stage_bufs: Dict[int, DeviceBuffer] = {}
        star = sc.ce_transport and sc.overlap  # copy-engine star: per-copy flags, no relay array
        if sc.ce_transport and world > 1:  # schedule (and star) flags
            ce_flag = DeviceBuffer(self.cuda_device, 4 * max(ce_slots(p, self.host_of), 64))
            ce_flag.zero()
            b.owned.append(ce_flag)
            mine["cflag"] = {rank: ce_flag.ipc_handle()} if world > 1 else {}
        elif sc.relay or sc.overlap:
            slots = relay_slots(p, self.host_of, self.chunk_bytes, chain=sc.relay, overlap=sc.overlap)
            if slots:
                relay_buf = DeviceBuffer(self.cuda_device, 4 * max(slots, 64))
                relay_buf.zero()
                b.owned.append(relay_buf)
                mine["relay"] = {rank: relay_buf.ipc_handle()} if world > 1 else {}
        if sc.staged:
            need = sorted({s for s, dsts, _r in p.lowered() if self.host_of[s] != rank and
                           any(self.host_of[d] == rank for d in dsts)})
            stage_bufs = {s: DeviceBuffer(self.cuda_device, p.shard_bytes(SRC, s)) for s in need}
            b.owned.extend(stage_bufs.values())
            stage_flag = DeviceBuffer(self.cuda_device, 4 * max(stage_slots(p, self.host_of, self.stage_chunk), 64))
            stage_flag.zero()
            b.owned.append(stage_flag)
            mine["stage"] = {s: x.ipc_handle() for s, x in stage_bufs.items()}
            mine["sflag"] = {rank: stage_flag.ipc_handle()}
        stream_sync()
        gathered = self._exchange(mine) if (sc.relay or sc.overlap or sc.staged or sc.ce_transport) else [mine] * world
        relay_remote: Dict[int, int] = {}
        ce_flags: Dict[int, int] = {rank: ce_flag.ptr} if ce_flag else {}
        stage_remote: Dict[Tuple[int, int], int] = {}
        stage_flags: Dict[int, int] = {rank: stage_flag.ptr} if stage_flag else {}
        for r, table in enumerate(gathered):
            if r == rank:
                continue
            for key, handles in table.items():
                for d, h in handles.items():
                    if key == "stage" and self.owner[d] != rank:
                        continue  # another GPU's staging for a source not held here
                    ptr = open_ipc(self.cuda_device, h)
                    b.opened.append(ptr)
                    if key == "relay":
                        relay_remote[r] = ptr
                    elif key == "cflag":
                        ce_flags[r] = ptr
                    elif key == "stage":
                        stage_remote[(d, r)] = ptr
                    else:
                        stage_flags[r] = ptr
        if sc.nccl:
            self._bind_nccl(pi, b)
            return
        if sc.staged:
            # pull-mode unpack from local staging buffers; this GPU's own
            # sources are pushed to the others by its copy engine
            src = {d: ptr for d, ptr in self.ptrs[sname].items() if self.owner[d] == rank}
            src.update({d: x.ptr for d, x in stage_bufs.items()})
            ex = Executor(p, self.cuda_device, src, self.ptrs[dname], self.local, PULL, self.chunk_bytes,
                          host_of=self.host_of, stage_chunk_bytes=self.stage_chunk, n_hosts=world,
                          stage_remote=stage_remote, stage_flags=stage_flags)
        else:
            relay_table = None
            if relay_buf is not None:
                relay_table = {d: (relay_buf.ptr if self.owner[d] == rank else relay_remote[self.owner[d]])
                               for d in range(n)}
            ex = Executor(p, self.cuda_device, self.ptrs[sname], self.ptrs[dname], self.local, self.mode,
                          self.chunk_bytes, host_of=self.host_of if self.hierarchical else None,
                          mc_ptrs=self.mc_tables.get(dname) if sc.multicast else None,
                          relay_flags=relay_table, relay_chain=sc.relay,
                          overlap_fanout=sc.overlap, ce_min_run_bytes=self.ce_min_run_bytes,
                          ce_transport=(3 if sc.relay and sc.ce_transport else 2 if sc.ce_hybrid
                                        else int(sc.ce_transport)),
                          n_hosts=world if ce_flag else 0,
                          ce_flags=ce_flags if ce_flag else None)
        if self.kernel is not None:
            ex.set_kernel(self.kernel)
        ex.set_flag_kernel(self.flag_kernel)
        b.executor = ex
        self.bindings[pi] = b
        if self.executors and pi < len(self.executors):
            self.executors[pi] = ex
        # Every rank must run the same barrier sequence: a phase has a fan-out
        # step if any rank has fan-out work in it.
        counts = self._exchange({"n": ex.fanout_items}) if world > 1 else [{"n": ex.fanout_items}]
        self.has_fanout[pi] = sum(c["n"] for c in counts) > 0

    def _bind_nccl(self, pi: int, b: "_Binding") -> None:
        """Scheme(nccl=True): staging for the remote sources this rank reads,
        the NCCL transfers, and the local pull executor that unpacks."""
        rank, world = self.rank, self.world
        p = self.plans[pi]
        sname, dname = self.bind[pi]
        need = self._remote_sources(pi)
        staging = {s: DeviceBuffer(self.cuda_device, p.shard_bytes(SRC, s)) for s in need}
        b.owned.extend(staging.values())
        # who reads what, identically on every rank
        readers: Dict[int, List[int]] = {}
        for s, dsts, _r in p.lowered():
            for d in dsts:
                if self.host_of[d] != self.host_of[s] and self.host_of[d] not in readers.setdefault(s, []):
                    readers[s].append(self.host_of[d])
        srcs = sorted(s for s in readers if readers[s])
        local_src = {d: buf for d, buf in self.buffers[sname].items() if self.owner[d] == rank}
        bcast = None
        sends, recvs = [], []
        if len(srcs) == 1 and sorted(readers[srcs[0]]) == [r for r in range(world) if r != self.host_of[srcs[0]]]:
            s0 = srcs[0]
            root = self.host_of[s0]
            if rank == root:
                t = _torch_bytes(local_src[s0].ptr, p.shard_bytes(SRC, s0))
            else:
                t = _torch_bytes(staging[s0].ptr, p.shard_bytes(SRC, s0))
            bcast = (t, root)
        else:
            for s in srcs:
                nb = p.shard_bytes(SRC, s)
                if self.host_of[s] == rank:
                    sends += [(_torch_bytes(local_src[s].ptr, nb), q) for q in sorted(readers[s])]
                elif rank in readers[s]:
                    recvs.append((_torch_bytes(staging[s].ptr, nb), self.host_of[s]))
        src = {d: buf.ptr for d, buf in local_src.items()}
        src.update({s: buf.ptr for s, buf in staging.items()})
        dst = {d: ptr for d, ptr in self.ptrs[dname].items() if self.owner[d] == rank}
        # flat pull: every local destination reads its slices straight from
        # local memory (own shards or staging), so no fan-out phase follows
        inner = Executor(p, self.cuda_device, src, dst, self.local, PULL, self.chunk_bytes)
        if self.kernel is not None:
            inner.set_kernel(self.kernel)
        b.executor = NcclStaged(inner, self.group, sends, recvs, bcast, local_src)
        self.bindings[pi] = b
        if self.executors and pi < len(self.executors):
            self.executors[pi] = b.executor
        self.has_fanout[pi] = False  # the pull executor writes every local replica itself

    def _unbind_phase(self, pi: int) -> None:
        stream_sync()
        self._collective_barrier()  # no rank still reads or writes this binding's buffers
        self.bindings[pi].free()
        self._collective_barrier()
        self.bindings[pi] = None

    # ---- reporting (bench, tests) -------------------------------------------

    def _phases_with(self, attr: str) -> List[int]:
        return [pi for pi, sc in enumerate(self.schemes) if getattr(sc, attr)]

    @property
    def relay_phases(self) -> List[int]:
        return self._phases_with("relay")

    @property
    def overlap_phases(self) -> List[int]:
        return self._phases_with("overlap")

    @property
    def staged_phases(self) -> List[int]:
        return self._phases_with("staged")

    @property
    def ce_phases(self) -> List[int]:
        return self._phases_with("ce_transport")

    @property
    def nccl_phases(self) -> List[int]:
        return self._phases_with("nccl")

    # ---- execution ------------------------------------------------------------

    def set_kernel(self, kernel: int, flag_kernel: Optional[int] = None) -> None:
        for e in self.executors:
            e.set_kernel(kernel)
            if flag_kernel is not None:
                e.set_flag_kernel(flag_kernel)

    def run_phase(self, i: int, stream=None, ctas: int = 0) -> None:
        """Phase i: direct copies, barrier, then (if any rank has some) the
        in-host fan-out from leader replicas and another barrier."""
        self.executors[i].launch(stream, ctas)
        self._finish_phase(i, stream, ctas)

    def _finish_phase(self, i: int, stream, ctas: int) -> None:
        if self.world > 1:
            self.barrier.launch(stream)
            if self.has_fanout[i]:
                self.bindings[i].executor.launch_fanout(stream, ctas)
                self.barrier.launch(stream)

    def run_phase_onload(self, i: int, host_ptrs: Dict[int, int], copy_stream, stream=None, ctas: int = 0,
                         chunk_bytes: int = 256 << 20) -> None:
        """Phase i with its local source shards onloaded from pinned host
        memory (host_ptrs: device -> pointer), H2D chunks overlapped with the
        copy kernels."""
        e = self.executors[i]
        sname = self.bind[i][0]
        key = (i, chunk_bytes, id(e))
        if getattr(self, "_onload_key", {}).get(i) != key:
            e.enable_onload({d: b.nbytes for d, b in self.buffers[sname].items()}, chunk_bytes)
            self._onload_key = {**getattr(self, "_onload_key", {}), i: key}
        e.launch_onload(host_ptrs, copy_stream, stream, ctas)
        self._finish_phase(i, stream, ctas)

    def run_phase_offload(self, i: int, host_ptrs: Dict[int, int], copy_stream, stream=None,
                          ctas: int = 0) -> None:
        """Phase i while its local source shards are parked in pinned host
        memory (host_ptrs: device -> pointer) on ``copy_stream``
        ("host-device (e.g., offload)"): the device->host copies
        and the reallocation kernels read the same shards concurrently."""
        sname = self.bind[i][0]
        self.executors[i].launch_offload({d: b.nbytes for d, b in self.buffers[sname].items()}, host_ptrs,
                                         copy_stream, stream)
        self.run_phase(i, stream, ctas)

    def close(self) -> None:
        stream_sync()
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier(group=self.group)  # no rank may still be storing into shared buffers
        for b in self.bindings:
            if b is not None:
                b.free()
        self.barrier.close()
        for p in self._opened:
            close_ipc(p)
        for pm in getattr(self, "_peer_mem", []):
            pm.close()
        for bufs in self.buffers.values():
            for b in bufs.values():
                b.free()
        self.flags.free()

    def relay_timeouts(self) -> int:
        """Relay / stage waits that gave up (bounded spins); nonzero = results invalid."""
        return sum(e.relay_timeouts() for e in self.executors)
