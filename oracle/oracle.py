"""TEST INFRASTRUCTURE — Python handle on the CPU oracle.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module. It wraps

* ``oracle/liboracle.so`` — the plain-C restatement of the reference
  algorithm (realloc_oracle.c, PAPER.md:500/515,
  reference model_arith.cpp:28-46 and cluster.cpp:23-30/95-101), and
* ``oracle/_ref/librlplan_ref.so`` — the reference's own
  proj/src/model_arith.cpp + cluster.cpp compiled where they lie
  (oracle/Makefile), used to pin the restatement and the product.

Arguments are duck-typed: anything with the attribute names of the
reference types (ModelSpec, ClusterSpec, DeviceMesh, Placement) works, so
this module never imports the product package.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_double, c_int, c_int32, c_int64, c_uint16, c_uint64, c_void_p
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "librlplan_ref.so")
MAX_DST = 64


class OrcModel(Structure):
    _fields_ = [("hidden", c_int64), ("ffn", c_int64), ("layers", c_int64), ("heads", c_int64),
                ("kv_heads", c_int64), ("vocab", c_int64), ("param_bytes", c_int64),
                ("has_output_head", c_int32)]


class OrcCluster(Structure):
    _fields_ = [("n_nodes", c_int32), ("gpus_per_node", c_int32), ("intra_bw", c_double), ("inter_bw", c_double)]


class OrcPlacement(Structure):
    _fields_ = [("node_offset", c_int32), ("node_count", c_int32), ("gpu_offset", c_int32),
                ("gpu_count", c_int32), ("dp", c_int32), ("tp", c_int32), ("pp", c_int32),
                ("qkv_layout", c_int32), ("gate_up_layout", c_int32), ("kv_layout", c_int32)]


class OrcOp(Structure):
    _fields_ = [("src", c_int32), ("n_dst", c_int32), ("dst", c_int32 * MAX_DST), ("layer_start", c_int64),
                ("layer_end", c_int64), ("slice", c_int32), ("slices", c_int32), ("replicated", c_int32),
                ("bytes", c_int64), ("part", c_int32)]


def _build_if_missing() -> None:
    if not os.path.exists(ORACLE_LIB):
        os.system(f"make -s -C {HERE} liboracle.so")


_build_if_missing()
_lib = ctypes.CDLL(ORACLE_LIB)
_lib.orc_param_count.restype = c_int64
_lib.orc_param_count.argtypes = [POINTER(OrcModel), c_int]
_lib.orc_stage_layer_map.argtypes = [c_int64, c_int, POINTER(c_int64), POINTER(c_int64)]
_lib.orc_plan.argtypes = [POINTER(OrcModel), POINTER(OrcPlacement), POINTER(OrcPlacement), POINTER(OrcCluster),
                          c_int, POINTER(OrcOp), c_int, POINTER(c_int), POINTER(OrcOp), c_int, POINTER(c_int),
                          POINTER(c_int64), POINTER(c_double)]
_lib.orc_shard_bytes.restype = c_int64
_lib.orc_shard_bytes.argtypes = [POINTER(OrcModel), POINTER(OrcPlacement), POINTER(OrcCluster), c_int]
_lib.orc_value.restype = c_uint16
_lib.orc_value.argtypes = [c_uint64, c_int64, c_int64]
_lib.orc_fill.argtypes = [POINTER(OrcModel), POINTER(OrcPlacement), POINTER(OrcCluster), c_int, c_uint64, c_void_p]
_lib.orc_execute.argtypes = [POINTER(OrcModel), POINTER(OrcPlacement), POINTER(OrcPlacement), POINTER(OrcCluster),
                             POINTER(OrcOp), c_int, POINTER(c_void_p), POINTER(c_void_p), c_int]


def _model(m) -> OrcModel:
    return OrcModel(m.hidden_size, m.intermediate_size, m.num_layers, m.num_attention_heads, m.num_kv_heads,
                    m.vocab_size, m.param_bytes, 1 if m.has_output_head else 0)


def _cluster(c) -> OrcCluster:
    return OrcCluster(c.n_nodes, c.gpus_per_node, c.intra_node_bw, c.inter_node_bw)


def _placement(p) -> OrcPlacement:
    m, s = p.mesh, p.strategy
    return OrcPlacement(m.node_offset, m.node_count, m.gpu_offset, m.gpu_count, s.dp, s.tp, s.pp,
                        getattr(p, "qkv_layout", 0), getattr(p, "gate_up_layout", 0), getattr(p, "kv_layout", 0))


# An op as a plain tuple: (src, dst tuple, (layer_start, layer_end, slice, slices, replicated, part), bytes);
# part: 0 every TP-split tensor, 1 all but k/v, 2 k/v only (DESIGN.md §3 G6)
OpTuple = Tuple[int, Tuple[int, ...], Tuple[int, int, int, int, bool, int], int]


def param_count(model, include_output_embedding: bool) -> int:
    return _lib.orc_param_count(ctypes.byref(_model(model)), int(include_output_embedding))


def stage_layer_map(num_layers: int, pp: int) -> Optional[List[Tuple[int, int]]]:
    n = max(pp, 1)
    a, b = (c_int64 * n)(), (c_int64 * n)()
    if _lib.orc_stage_layer_map(num_layers, pp, a, b):
        return None
    return [(a[i], b[i]) for i in range(pp)]


def _op_tuple(o: OrcOp) -> OpTuple:
    return (o.src, tuple(o.dst[: o.n_dst]),
            (o.layer_start, o.layer_end, o.slice, o.slices, bool(o.replicated), o.part), o.bytes)


def plan(model, src, dst, cluster, policy: int = 0):
    """SPEC plan_param_realloc restated. Returns (ops, local_ops, total_bytes,
    est_time) or None when a placement is invalid."""
    cap = 1 << 14
    ops, loc = (OrcOp * cap)(), (OrcOp * cap)()
    n, nl = c_int(), c_int()
    tb, et = c_int64(), c_double()
    rc = _lib.orc_plan(ctypes.byref(_model(model)), ctypes.byref(_placement(src)), ctypes.byref(_placement(dst)),
                       ctypes.byref(_cluster(cluster)), policy, ops, cap, ctypes.byref(n), loc, cap,
                       ctypes.byref(nl), ctypes.byref(tb), ctypes.byref(et))
    if rc:
        return None
    return ([_op_tuple(ops[i]) for i in range(n.value)], [_op_tuple(loc[i]) for i in range(nl.value)],
            tb.value, et.value)


def shard_bytes(model, placement, cluster, dev: int) -> int:
    return _lib.orc_shard_bytes(ctypes.byref(_model(model)), ctypes.byref(_placement(placement)),
                                ctypes.byref(_cluster(cluster)), dev)


def value(seed: int, tensor: int, index: int) -> int:
    return _lib.orc_value(seed, tensor, index)


def fill(model, placement, cluster, dev: int, seed: int) -> np.ndarray:
    """Expected shard of `dev` as uint16 (bf16 bits); padding bytes are zero."""
    n = shard_bytes(model, placement, cluster, dev)
    buf = np.zeros(n // 2, dtype=np.uint16)
    if n:
        rc = _lib.orc_fill(ctypes.byref(_model(model)), ctypes.byref(_placement(placement)),
                           ctypes.byref(_cluster(cluster)), dev, seed, buf.ctypes.data)
        assert rc == 0
    return buf


_lib.orc_fill_range.argtypes = [POINTER(OrcModel), POINTER(OrcPlacement), POINTER(OrcCluster), c_int, c_uint64,
                                c_int64, c_int64, c_void_p, c_int]
_lib.orc_check_range.argtypes = [POINTER(OrcModel), POINTER(OrcPlacement), POINTER(OrcCluster), c_int, c_uint64,
                                 c_int64, c_int64, c_void_p, c_int, POINTER(c_int64), POINTER(c_int64)]
SEED_SPECIAL = 1 << 62  # special-value mode (ORC_SEED_SPECIAL)


def fill_range_into(model, placement, cluster, dev: int, seed: int, offset: int, nbytes: int, ptr: int,
                    threads: int = 0) -> None:
    """Write bytes [offset, offset + nbytes) of the expected shard of `dev` to
    host address `ptr` (padding zero), with `threads` threads (0 = all)."""
    rc = _lib.orc_fill_range(ctypes.byref(_model(model)), ctypes.byref(_placement(placement)),
                             ctypes.byref(_cluster(cluster)), dev, seed, offset, nbytes, ptr,
                             threads or (os.cpu_count() or 1))
    assert rc == 0, "orc_fill_range: bad window"


def fill_mt(model, placement, cluster, dev: int, seed: int, threads: int = 0) -> np.ndarray:
    """fill() computed with several threads (multi-GB shards)."""
    n = shard_bytes(model, placement, cluster, dev)
    buf = np.empty(n // 2, dtype=np.uint16)
    if n:
        fill_range_into(model, placement, cluster, dev, seed, 0, n, buf.ctypes.data, threads)
    return buf


def check_range(model, placement, cluster, dev: int, seed: int, offset: int, nbytes: int, ptr: int,
                threads: int = 0) -> Tuple[int, int]:
    """Compare nbytes at host address `ptr` with the expected shard window at
    `offset`: (mismatching bf16 elements, first mismatching element of the
    window or -1). Runs without the GIL (ctypes), so a caller may overlap it
    with a device->host copy of the next window."""
    bad, first = c_int64(), c_int64()
    rc = _lib.orc_check_range(ctypes.byref(_model(model)), ctypes.byref(_placement(placement)),
                              ctypes.byref(_cluster(cluster)), dev, seed, offset, nbytes, ptr,
                              threads or (os.cpu_count() or 1), ctypes.byref(bad), ctypes.byref(first))
    assert rc == 0, "orc_check_range: bad window"
    return bad.value, first.value


def _ops_array(ops: Sequence[OpTuple]):
    arr = (OrcOp * max(1, len(ops)))()
    for i, (s, d, (lo, hi, k, G, rep, part), b) in enumerate(ops):
        arr[i].src, arr[i].n_dst = s, len(d)
        for j, x in enumerate(d):
            arr[i].dst[j] = x
        arr[i].layer_start, arr[i].layer_end = lo, hi
        arr[i].slice, arr[i].slices, arr[i].replicated, arr[i].bytes = k, G, int(rep), b
        arr[i].part = part
    return arr


def execute(model, src, dst, cluster, ops: Sequence[OpTuple], src_bufs: Sequence[Optional[np.ndarray]],
            dst_bufs: Sequence[Optional[np.ndarray]], threads: int = 1) -> None:
    """CPU reallocation: run `ops` (remote + local) on host numpy buffers."""
    n = cluster.n_nodes * cluster.gpus_per_node
    sp, dp = (c_void_p * n)(), (c_void_p * n)()
    for i in range(n):
        sp[i] = src_bufs[i].ctypes.data if src_bufs[i] is not None else None
        dp[i] = dst_bufs[i].ctypes.data if dst_bufs[i] is not None else None
    arr = _ops_array(ops)
    _lib.orc_execute(ctypes.byref(_model(model)), ctypes.byref(_placement(src)), ctypes.byref(_placement(dst)),
                     ctypes.byref(_cluster(cluster)), arr, len(ops), sp, dp, threads)


def _mesh_devices(placement, cluster) -> List[int]:
    m = placement.mesh
    return [(m.node_offset + n) * cluster.gpus_per_node + m.gpu_offset + g
            for n in range(m.node_count) for g in range(m.gpu_count)]


def _kv_slices(model, placement) -> int:
    """DESIGN.md §3 G6: distinct K/V slices over the TP ranks."""
    tp = placement.strategy.tp
    return model.num_kv_heads if getattr(placement, "kv_layout", 0) == 1 and tp > model.num_kv_heads else tp


def _units(model, placement, cluster, G: int, Gkv: int = 0):
    """Per device: set of shard units it holds — (ext_layer, k) for each of the
    G finest slices of the split tensors and (ext_layer, 'rep') for the
    replicated ones (SPEC.md:596 finest common slicing). With Gkv (K/V
    carried separately, G6), k and v are units (layer, 'kv', k) of the Gkv
    finest K/V slices and the (ext_layer, k) units exclude them."""
    L = model.num_layers
    s = placement.strategy
    kv = _kv_slices(model, placement)
    stages = stage_layer_map(L, s.pp)
    devs = _mesh_devices(placement, cluster)
    out = {}
    for idx, d in enumerate(devs):
        tp_r, pp_r = idx % s.tp, idx // (s.tp * s.dp)
        lo = -1 if pp_r == 0 else stages[pp_r][0]
        hi = L + 1 if pp_r == s.pp - 1 else stages[pp_r][1]
        units = set()
        for e in range(lo, hi):
            has_split = e != L or model.has_output_head
            has_rep = e != -1
            if has_split:
                per = G // s.tp
                units.update((e, k) for k in range(tp_r * per, (tp_r + 1) * per))
            if has_rep:
                units.add((e, "rep"))
            if Gkv and 0 <= e < L:
                mine, per_kv = tp_r * kv // s.tp, Gkv // kv
                units.update((e, "kv", k) for k in range(mine * per_kv, (mine + 1) * per_kv))
        out[d] = units
    return out


def replay(model, src, dst, cluster, ops: Sequence[OpTuple], local_ops: Sequence[OpTuple]) -> Optional[str]:
    """SPEC.md:577 / SPEC.md:679 set-reconstruction replay oracle.

    Replays ops + local ops over simulated shard sets: every source must hold
    what it sends, and each destination must end with exactly its
    requirement — no missing, no extra, no duplicate units. Returns None on
    success, else a description of the first discrepancy."""
    G = src.strategy.tp * dst.strategy.tp // np.gcd(src.strategy.tp, dst.strategy.tp)
    e1, e2 = _kv_slices(model, src), _kv_slices(model, dst)
    Gkv = e1 * e2 // np.gcd(e1, e2) if (e1, e2) != (src.strategy.tp, dst.strategy.tp) else 0
    held = _units(model, src, cluster, G, Gkv)
    need = _units(model, dst, cluster, G, Gkv)
    got = {d: [] for d in need}
    for (s, dsts, (lo, hi, k, slices, rep, part), _b) in list(ops) + list(local_ops):
        units = []
        for e in range(lo, hi):
            if rep:
                if e != -1:  # the embedding has no replicated tensor
                    units.append((e, "rep"))
            elif part == 2:
                if 0 <= e < model.num_layers:
                    units.append((e, "kv", k))
            else:
                if e == model.num_layers and not model.has_output_head:
                    continue
                units.append((e, k))
        for u in units:
            if u not in held.get(s, set()):
                return f"source {s} does not hold {u}"
        for d in dsts:
            if d not in got:
                return f"destination {d} is not in the destination placement"
            got[d].extend(units)
    for d, req in need.items():
        if len(got[d]) != len(set(got[d])):
            return f"device {d} receives a unit twice"
        if set(got[d]) != req:
            missing, extra = req - set(got[d]), set(got[d]) - req
            return f"device {d}: missing {sorted(missing, key=str)[:4]} extra {sorted(extra, key=str)[:4]}"
    return None


# ---- the reference's own C++ (oracle/_ref) ------------------------------------

class Reference:
    """ctypes view of oracle/_ref/librlplan_ref.so (reference sources compiled as-is)."""

    def __init__(self, path: str = REF_LIB):
        self.lib = ctypes.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_param_count.argtypes = [POINTER(c_int64), c_int, c_int, POINTER(c_int64)]
        L.ref_static_param_bytes.argtypes = [POINTER(c_int64), c_int, POINTER(c_int64)]
        L.ref_flops.argtypes = [POINTER(c_int64), c_int, c_int, c_int64, c_int64, POINTER(c_double)]
        L.ref_kv_cache_bytes.restype = c_int64
        L.ref_kv_cache_bytes.argtypes = [POINTER(c_int64), c_int, c_int64, c_int64]
        L.ref_logits_bytes.restype = c_int64
        L.ref_logits_bytes.argtypes = [c_int64] * 4
        L.ref_enumerate_meshes.argtypes = [c_int, c_int, POINTER(c_int), c_int]
        L.ref_validate_mesh.argtypes = [c_int, c_int, POINTER(c_int)]
        L.ref_mesh_devices.argtypes = [c_int, c_int, POINTER(c_int), POINTER(c_int)]
        L.ref_overlap.argtypes = [c_int, c_int, POINTER(c_int), POINTER(c_int)]
        L.ref_link_bandwidth.argtypes = [c_int, c_int, c_int, c_int, POINTER(c_double)]
        L.ref_mesh_to_string.argtypes = [c_int, c_int, POINTER(c_int), ctypes.c_char_p, c_int]
        L.ref_mesh_from_string.argtypes = [c_int, c_int, ctypes.c_char_p, POINTER(c_int)]

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_LIB)

    @staticmethod
    def _dims(m):
        return (c_int64 * 10)(m.hidden_size, m.intermediate_size, m.num_layers, m.num_attention_heads,
                              m.num_kv_heads, m.vocab_size, m.max_position_embeddings, m.param_bytes,
                              m.grad_bytes, m.optimizer_bytes_per_param)

    def error(self) -> str:
        return self.lib.ref_last_error().decode()

    def param_count(self, m, include: bool):
        out = c_int64()
        rc = self.lib.ref_param_count(self._dims(m), int(m.has_output_head), int(include), ctypes.byref(out))
        return None if rc else out.value

    def static_param_bytes(self, m):
        out = (c_int64 * 3)()
        rc = self.lib.ref_static_param_bytes(self._dims(m), int(m.has_output_head), out)
        return None if rc else tuple(out)

    def flops(self, m, backward: bool, tokens: int, ctx: int):
        out = c_double()
        rc = self.lib.ref_flops(self._dims(m), int(m.has_output_head), int(backward), tokens, ctx, ctypes.byref(out))
        return None if rc else out.value

    def kv_cache_bytes(self, m, batch, seq):
        return self.lib.ref_kv_cache_bytes(self._dims(m), int(m.has_output_head), batch, seq)

    def logits_bytes(self, v, b, c, e):
        return self.lib.ref_logits_bytes(v, b, c, e)

    def enumerate_meshes(self, nodes: int, gpus: int) -> List[Tuple[int, int, int, int]]:
        cap = 4096
        buf = (c_int * (4 * cap))()
        n = self.lib.ref_enumerate_meshes(nodes, gpus, buf, cap)
        return [tuple(buf[4 * i: 4 * i + 4]) for i in range(n)]

    def validate_mesh(self, nodes, gpus, mesh) -> Optional[str]:
        rc = self.lib.ref_validate_mesh(nodes, gpus, (c_int * 4)(*mesh))
        return self.error() if rc else None

    def mesh_devices(self, nodes, gpus, mesh) -> List[int]:
        out = (c_int * 4096)()
        n = self.lib.ref_mesh_devices(nodes, gpus, (c_int * 4)(*mesh), out)
        return list(out[:n])

    def overlap(self, nodes, gpus, a, b) -> bool:
        return bool(self.lib.ref_overlap(nodes, gpus, (c_int * 4)(*a), (c_int * 4)(*b)))

    def link_bandwidth(self, nodes, gpus, a, b):
        out = c_double()
        rc = self.lib.ref_link_bandwidth(nodes, gpus, a, b, ctypes.byref(out))
        return None if rc else out.value

    def mesh_to_string(self, nodes, gpus, mesh) -> str:
        buf = ctypes.create_string_buffer(128)
        self.lib.ref_mesh_to_string(nodes, gpus, (c_int * 4)(*mesh), buf, 128)
        return buf.value.decode()

    def mesh_from_string(self, nodes, gpus, text):
        out = (c_int * 4)()
        rc = self.lib.ref_mesh_from_string(nodes, gpus, text.encode(), out)
        return (None, self.error()) if rc else (tuple(out), None)


# ---- inter-call data transfer --------------------------------

DATA_TENSOR = 0x7fff0000
_lib.orc_plan_data.argtypes = [POINTER(OrcPlacement), POINTER(OrcPlacement), POINTER(OrcCluster), c_int, c_int64,
                               POINTER(OrcOp), c_int, POINTER(c_int), POINTER(OrcOp), c_int, POINTER(c_int),
                               POINTER(c_int64), POINTER(c_double)]
_lib.orc_data_shard_bytes.restype = c_int64
_lib.orc_data_shard_bytes.argtypes = [POINTER(OrcPlacement), POINTER(OrcCluster), c_int, c_int, c_int64]
_lib.orc_data_fill.argtypes = [POINTER(OrcPlacement), POINTER(OrcCluster), c_int, c_int, c_int64, c_uint64, c_void_p]
_lib.orc_data_execute.argtypes = [POINTER(OrcPlacement), POINTER(OrcPlacement), POINTER(OrcCluster), c_int64,
                                  POINTER(OrcOp), c_int, POINTER(c_void_p), POINTER(c_void_p)]
_lib.orc_data_execute_mt.argtypes = [POINTER(OrcPlacement), POINTER(OrcPlacement), POINTER(OrcCluster), c_int64,
                                     POINTER(OrcOp), c_int, POINTER(c_void_p), POINTER(c_void_p), c_int]


def plan_data(producer, consumer, cluster, data_bytes_per_dp_shard: int, policy: int = 0):
    cap = 1 << 12
    ops, loc = (OrcOp * cap)(), (OrcOp * cap)()
    n, nl = c_int(), c_int()
    tb, et = c_int64(), c_double()
    rc = _lib.orc_plan_data(ctypes.byref(_placement(producer)), ctypes.byref(_placement(consumer)),
                            ctypes.byref(_cluster(cluster)), policy, data_bytes_per_dp_shard, ops, cap,
                            ctypes.byref(n), loc, cap, ctypes.byref(nl), ctypes.byref(tb), ctypes.byref(et))
    if rc:
        return None
    return ([_op_tuple(ops[i]) for i in range(n.value)], [_op_tuple(loc[i]) for i in range(nl.value)],
            tb.value, et.value)


def data_shard_bytes(placement, cluster, dev: int, producer: bool, total_bytes: int) -> int:
    return _lib.orc_data_shard_bytes(ctypes.byref(_placement(placement)), ctypes.byref(_cluster(cluster)), dev,
                                     int(producer), total_bytes)


def data_fill(placement, cluster, dev: int, producer: bool, total_bytes: int, seed: int) -> np.ndarray:
    n = data_shard_bytes(placement, cluster, dev, producer, total_bytes)
    buf = np.zeros(n // 2, dtype=np.uint16)
    if n:
        assert _lib.orc_data_fill(ctypes.byref(_placement(placement)), ctypes.byref(_cluster(cluster)), dev,
                                  int(producer), total_bytes, seed, buf.ctypes.data) == 0
    return buf


def data_execute(producer, consumer, cluster, total_bytes: int, ops, src_bufs, dst_bufs, threads: int = 1) -> None:
    n = cluster.n_nodes * cluster.gpus_per_node
    sp, dp = (c_void_p * n)(), (c_void_p * n)()
    for i in range(n):
        sp[i] = src_bufs[i].ctypes.data if src_bufs[i] is not None else None
        dp[i] = dst_bufs[i].ctypes.data if dst_bufs[i] is not None else None
    arr = _ops_array(ops)
    assert _lib.orc_data_execute_mt(ctypes.byref(_placement(producer)), ctypes.byref(_placement(consumer)),
                                    ctypes.byref(_cluster(cluster)), total_bytes, arr, len(ops), sp, dp,
                                    threads) == 0


def replay_data(producer, consumer, cluster, data_bytes_per_dp_shard: int, ops, local_ops):
    """SPEC.md:586 replay: each consumer device ends with exactly its DP
    group's slices; every source (right DP rank) holds what it sends."""
    G = int(np.lcm(producer.strategy.dp, consumer.strategy.dp))

    def ranks(p):
        devs = _mesh_devices(p, cluster)
        s = p.strategy
        return {d: (i // (s.tp * s.dp), (i // s.tp) % s.dp) for i, d in enumerate(devs)}
    pr, cr = ranks(producer), ranks(consumer)
    got = {d: [] for d in cr}
    for (s, dsts, (lo, hi, k, slices, rep, _part), _b) in list(ops) + list(local_ops):
        if slices != G or rep or s not in pr:
            return f"bad payload from {s}"
        pp_r, dp_r = pr[s]
        if k // (G // producer.strategy.dp) != dp_r:
            return f"source {s} does not hold slice {k}"
        for d in dsts:
            if d not in got:
                return f"{d} is not a consumer"
            got[d].append(k)
    per = G // consumer.strategy.dp
    for d, ks in got.items():
        want = list(range(cr[d][1] * per, (cr[d][1] + 1) * per))
        if sorted(ks) != want:
            return f"consumer {d} got {sorted(ks)} want {want}"
    return None
