"""Measured B200 cost model of a reallocation.

The reference's simulator gives a param_realloc node the SPEC estimate
``est_time = max over sources of sum(bytes / bandwidth)`` (SPEC.md:572,
SPEC.md:420-428). This module replaces that with the time this executor
actually takes on B200, from the same lowered work the kernels run:

* per GPU, HBM bytes (every copy reads its source once and writes each
  local destination; hierarchical fan-out included) at the measured
  effective copy bandwidth of the TMA bulk kernel;
* per GPU, link bytes in and out at the measured NVLink rate of the peer
  store path (or the multicast rate for multicast payloads), except the
  bytes of copy-engine runs (rr_exec_options.ce_min_run_bytes), which move
  at the measured copy-engine rate on the same link;
* phases serialise, GPUs run in parallel: time = max over GPUs of
  max(HBM time, link time) per phase, plus a fixed launch/barrier cost.
* offload / onload of parked parameters (SPEC.md:423 prices them at
  ``bytes / host_to_device_bw``) at the measured host-link rate per GPU; a
  pipelined onload overlaps phase 0, so that phase takes the longer of the
  two.

* the copy-engine transport (r02) by the library's own schedule simulation
  (`estimate_best` picks the fastest scheme, as the bind-time probe does by
  measurement).

Constants are the r01/r02 measurements (profiles/).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Optional, Sequence

from .rlplan import ReallocPlan


@dataclass(frozen=True)
class B200Profile:
    hbm_copy_gbs: float = 6340.0        # read+write bytes/s of rr_bulk_kernel (7B tp8->dp8 forward, 1 GPU)
    nvlink_push_gbs: float = 708.0      # per GPU per direction, SM peer stores (2/4 GPUs, all-to-all)
    nvlink_mc_gbs: float = 565.0        # per receiving GPU, NVLS multimem.st (4 GPUs)
    nvlink_ce_gbs: float = 777.0        # per GPU per direction, whole copy-engine copies, pairwise (2/4 GPUs)
    nvlink_ce_rot_gbs: float = 771.0    # copy-engine rotation rounds (staged gather), 4 GPUs
    launch_us: float = 8.0              # kernel launch + dynamic-scheduler tail
    barrier_us: float = 12.0            # cross-GPU flag barrier
    host_link_gbs: float = 55.6         # pinned host <-> HBM per GPU, either direction (r01 ce_probe h2d/*)


def host_transfer_seconds(nbytes_per_gpu: int, profile: B200Profile = B200Profile()) -> float:
    """Duration of an offload or onload node that moves
    ``nbytes_per_gpu`` between pinned host memory and each GPU's HBM (every
    GPU has its own host link)."""
    return nbytes_per_gpu / (profile.host_link_gbs * 1e9)


def estimate_best(plan: ReallocPlan, host_of: Optional[Sequence[int]] = None,
                  profile: B200Profile = B200Profile()) -> Dict[str, float]:
    """The fastest delivery scheme by this model (what the bind-time probe
    measures at run time): SM peer stores with copy-engine runs, the
    pipelined relay, the staged gather, and the copy-engine transport
    (schedule makespan, r02), with the scheme's name under "scheme"."""
    est = {"push": estimate_seconds(plan, host_of, profile)}
    n = plan.cluster.device_count()
    host = list(host_of) if host_of is not None else list(range(n))
    if len(set(host)) > 1:
        est["relay"] = estimate_seconds(plan, host_of, profile, relay=True)
        est["staged"] = estimate_seconds(plan, host_of, profile, staged=True)
        est["ce_transport"] = estimate_seconds(plan, host_of, profile, ce_transport=True)
    name = min(est, key=lambda k: est[k]["seconds"])
    return {**est[name], "scheme": name}


def estimate_seconds(plan: ReallocPlan, host_of: Optional[Sequence[int]] = None,
                     profile: B200Profile = B200Profile(), multicast: bool = False,
                     relay: bool = False, onload: bool = False, copy_engine: bool = True,
                     staged: bool = False, ce_transport: bool = False) -> Dict[str, float]:
    """Estimated execution time of `plan` with plan device d hosted on GPU
    host_of[d] (default: one GPU per plan device). `relay`: payloads reaching
    >= 2 other GPUs use the pipelined relay (one copy in and out per GPU,
    fan-out fused into phase 0). `onload`: the source shards arrive from
    pinned host memory pipelined with phase 0 (rr_exec_launch_onload).
    `copy_engine`: ranges laid out identically on both sides move as
    copy-engine runs (the executor default; not combined with relay or
    multicast here). `staged`: the remote bytes move as a staged gather
    (copy-engine rotation rounds into staging buffers, then an unpack that
    reads them once more from HBM). `ce_transport`: every remote piece moves
    by copy engine as merged 2D/3D copies following the library's schedule
    (its simulated makespan, rr_plan_ce_schedule), the in-host fan-out
    overlapped (copy-engine star)."""
    if ce_transport:
        from .runtime import ce_transport_estimate
        n = plan.cluster.device_count()
        host = list(host_of) if host_of is not None else list(range(n))
        if len(set(host)) > 1:
            ce, _sm = ce_transport_estimate(plan, host, star=True)
            fixed = (profile.launch_us + profile.barrier_us) * 1e-6
            base = estimate_seconds(plan, host_of, profile, copy_engine=False)
            return {**base, "seconds": ce + fixed, "phase0_s": ce, "fanout_s": 0.0}
    n = plan.cluster.device_count()
    host = list(host_of) if host_of is not None else list(range(n))
    hosts = sorted(set(host))
    hbm = {h: 0 for h in hosts}
    fan = {h: 0 for h in hosts}
    egress = {h: 0 for h in hosts}
    ingress = {h: 0 for h in hosts}
    mc_in = {h: 0 for h in hosts}
    for s, dsts, rects in plan.lowered():
        b = sum(r[2] * r[5] for r in rects)
        hs = host[s]
        groups: Dict[int, list] = {}
        for d in dsts:
            groups.setdefault(host[d], []).append(d)
        local = groups.get(hs, [])
        hbm[hs] += b * (1 + len(local))      # one read, one write per local destination
        remote = [h for h in groups if h != hs]
        if relay and len(remote) >= 2:
            chain = sorted(remote, key=lambda h: (h - hs) % (max(hosts) + 1))
            egress[hs] += b
            for k, h in enumerate(chain):
                ingress[h] += b
                egress[h] += b if k + 1 < len(chain) else 0
                hbm[h] += b * (1 + len(groups[h]))  # leader written, read once, other replicas written
            continue
        use_mc = multicast and set(groups) == set(hosts) and len(remote) > 0
        if use_mc:
            egress[hs] += b
            for h in groups:
                mc_in[h] += b
        else:
            egress[hs] += b * len(remote)
            for h in remote:
                ingress[h] += b
        for h in remote:
            extra = len(groups[h]) - 1       # hierarchical fan-out inside host h
            hbm[h] += b                      # the leader replica is written once
            fan[h] += b * (1 + extra) if extra else 0  # read the leader, write the others
    # copy-engine runs: their bytes leave the SM push totals and take the
    # copy-engine rate on the same link
    ce_out = {h: 0 for h in hosts}
    ce_in = {h: 0 for h in hosts}
    if copy_engine and not relay and not multicast and len(hosts) > 1:
        for h in hosts:
            local = [d for d in range(n) if host[d] == h]
            for (s, d, _so, _do, nb) in plan.ce_runs(local, host):
                ce_out[h] += nb
                ce_in[host[d]] += nb
        for h in hosts:
            egress[h] = max(0, egress[h] - ce_out[h])
            ingress[h] = max(0, ingress[h] - ce_in[h])

    if staged and len(hosts) > 1:
        # the staged gather moves WHOLE source shards to every host that
        # reads any of their bytes (rr_plan_stage_slots), not just the bytes
        # read; staging is written, then read back by the unpack, which
        # writes every local replica
        reads = {(s, host[d]) for s, dsts, _r in plan.lowered() for d in dsts if host[d] != host[s]}
        ingress = {h: 0 for h in hosts}
        egress = {h: 0 for h in hosts}
        for s, h in reads:
            ingress[h] += plan.shard_bytes(0, s)
            egress[host[s]] += plan.shard_bytes(0, s)
        for h in hosts:
            hbm[h] += 2 * ingress[h] + fan[h]
            fan[h] = 0

    def link_s(h: int) -> float:
        if staged:
            return max(egress[h], ingress[h]) / (profile.nvlink_ce_rot_gbs * 1e9)
        out = egress[h] / (profile.nvlink_push_gbs * 1e9) + ce_out[h] / (profile.nvlink_ce_gbs * 1e9)
        inn = ingress[h] / (profile.nvlink_push_gbs * 1e9) + ce_in[h] / (profile.nvlink_ce_gbs * 1e9)
        return max(out, inn) + mc_in[h] / (profile.nvlink_mc_gbs * 1e9)

    t_phase0 = max(max(hbm[h] / (profile.hbm_copy_gbs * 1e9), link_s(h)) for h in hosts)
    onload_s = 0.0
    if onload:
        src_bytes = {h: 0 for h in hosts}
        for d in plan.devices(0):
            src_bytes[host[d]] += plan.shard_bytes(0, d)
        onload_s = max(host_transfer_seconds(b, profile) for b in src_bytes.values())
        t_phase0 = max(t_phase0, onload_s)
    t_phase1 = max(fan[h] / (profile.hbm_copy_gbs * 1e9) for h in hosts)
    multi = len(hosts) > 1
    fixed = profile.launch_us * 1e-6 * (2 if t_phase1 > 0 else 1)
    if multi:
        fixed += profile.barrier_us * 1e-6 * (2 if t_phase1 > 0 else 1)
    total = t_phase0 + t_phase1 + fixed
    return {"seconds": total, "phase0_s": t_phase0, "fanout_s": t_phase1, "onload_s": onload_s,
            "spec_est_time_s": plan.est_time,
            "max_link_bytes": max(max(egress[h] + ce_out[h], ingress[h] + ce_in[h]) + mc_in[h] for h in hosts),
            "max_hbm_bytes": max(hbm[h] for h in hosts)}
