"""ctypes binding of librrealloc.so (the C ABI declared in include/rr_realloc.h).

The shared library is the product: planner, layout contract and the sm_100a
kernels. There is deliberately no fallback — if the library is missing the
import fails loudly (build it with ``python -c "import __graft_entry__ as g;
g.build()"`` or ``make -C paper_2406_14088_b200/csrc``).
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_char, c_char_p, c_double, c_float, c_int, c_int32,
                    c_int64, c_size_t, c_uint16, c_uint64, c_void_p)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "librrealloc.so")

RR_OK, RR_EINVAL, RR_ECUDA, RR_ENOMEM, RR_EUNSUPPORTED, RR_ETIMEOUT, RR_ERANGE = range(7)


class RrModel(Structure):
    _fields_ = [("name", c_char_p), ("hidden_size", c_int64), ("intermediate_size", c_int64),
                ("num_layers", c_int64), ("num_attention_heads", c_int64), ("num_kv_heads", c_int64),
                ("vocab_size", c_int64), ("max_position_embeddings", c_int64), ("param_bytes", c_int64),
                ("grad_bytes", c_int64), ("optimizer_bytes_per_param", c_int64),
                ("has_output_head", c_int32)]


class RrCluster(Structure):
    _fields_ = [("n_nodes", c_int32), ("gpus_per_node", c_int32), ("mem_per_device", c_int64),
                ("intra_node_bw", c_double), ("inter_node_bw", c_double), ("host_to_device_bw", c_double)]


class RrMesh(Structure):
    _fields_ = [("node_offset", c_int32), ("node_count", c_int32), ("gpu_offset", c_int32),
                ("gpu_count", c_int32)]


class RrPlacement(Structure):
    _fields_ = [("mesh", RrMesh), ("dp", c_int32), ("tp", c_int32), ("pp", c_int32),
                ("n_microbatches", c_int32), ("qkv_layout", c_int32), ("gate_up_layout", c_int32),
                ("kv_layout", c_int32)]


class RrShard(Structure):
    _fields_ = [("layer_start", c_int64), ("layer_end", c_int64), ("tp_rank", c_int32),
                ("tp_degree", c_int32), ("replicated", c_int32), ("part", c_int32)]


class RrOp(Structure):
    _fields_ = [("src", c_int32), ("n_dst", c_int32), ("dst", POINTER(c_int32)), ("payload", RrShard),
                ("bytes", c_int64)]


class RrExecOptions(Structure):
    _fields_ = [("mode", c_int32), ("chunk_bytes", c_int64), ("host_of", POINTER(c_int32)),
                ("mc_bufs", POINTER(c_void_p)), ("relay_flags", POINTER(c_void_p)), ("relay_chain", c_int32),
                ("overlap_fanout", c_int32), ("ce_min_run_bytes", c_int64), ("stage_chunk_bytes", c_int64),
                ("n_hosts", c_int32), ("stage_remote", POINTER(c_void_p)), ("stage_flags", POINTER(c_void_p)),
                ("ce_transport", c_int32), ("ce_flags", POINTER(c_void_p))]


_P = c_void_p
_SIGNATURES = {
    "rr_exec_create_ex": (c_int, [_P, c_int, c_int, POINTER(_P), POINTER(_P), c_int, POINTER(c_int32),
                                  POINTER(RrExecOptions), POINTER(_P)]),
    "rr_plan_relay_slots": (c_int, [_P, POINTER(c_int32), c_int64, c_int, c_int, POINTER(c_int64)]),
    "rr_exec_relay_timeouts": (c_int, [_P, POINTER(c_int64)]),
    "rr_exec_kernel_count": (c_int, [_P, POINTER(c_int), POINTER(c_int)]),
    "rr_exec_phase_kernels": (c_int, [_P, c_int, POINTER(c_int), POINTER(c_int)]),
    "rr_exec_ce_runs": (c_int, [_P, POINTER(c_int), POINTER(c_int64)]),
    "rr_exec_stage_pushes": (c_int, [_P, POINTER(c_int), POINTER(c_int64)]),
    "rr_plan_stage_slots": (c_int, [_P, POINTER(c_int32), c_int64, POINTER(c_int64)]),
    "rr_plan_ce_runs": (c_int, [_P, c_int, POINTER(c_int32), POINTER(c_int32), c_int64, POINTER(c_int64), c_int,
                                POINTER(c_int)]),
    "rr_plan_ce_slots": (c_int, [_P, POINTER(c_int32), POINTER(c_int64)]),
    "rr_plan_ce_schedule": (c_int, [_P, POINTER(c_int32), POINTER(c_double), c_int, POINTER(c_int)]),
    "rr_plan_ce_copies": (c_int, [_P, c_int, POINTER(c_int32), POINTER(c_int32), POINTER(c_int64), c_int,
                                  POINTER(c_int)]),
    "rr_mcast_supported": (c_int, [c_int, POINTER(c_int)]),
    "rr_mcast_create": (c_int, [c_int, c_size_t, c_int, POINTER(c_int), POINTER(c_size_t), POINTER(_P)]),
    "rr_mcast_import": (c_int, [c_int, c_int, c_size_t, c_int, POINTER(_P)]),
    "rr_mcast_bind": (c_int, [_P, POINTER(_P), POINTER(_P)]),
    "rr_mcast_size": (c_int, [_P, POINTER(c_size_t)]),
    "rr_mcast_destroy": (None, [_P]),
    "rr_mcast_export_member": (c_int, [_P, POINTER(c_int)]),
    "rr_peer_mem_import": (c_int, [c_int, c_int, c_size_t, POINTER(_P), POINTER(_P)]),
    "rr_peer_mem_close": (None, [_P]),
    "rr_last_error": (c_char_p, []),
    "rr_abi_version": (c_int, []),
    "rr_model_validate": (c_int, [POINTER(RrModel)]),
    "rr_param_count": (c_int, [POINTER(RrModel), c_int, POINTER(c_int64)]),
    "rr_natural_param_count": (c_int, [POINTER(RrModel), POINTER(c_int64)]),
    "rr_flops": (c_int, [POINTER(RrModel), c_int, c_int64, c_int64, POINTER(c_double)]),
    "rr_layer_flops_fwd": (c_int, [POINTER(RrModel), c_int64, c_int64, POINTER(c_double)]),
    "rr_kv_cache_bytes": (c_int, [POINTER(RrModel), c_int64, c_int64, POINTER(c_int64)]),
    "rr_logits_bytes": (c_int, [c_int64, c_int64, c_int64, c_int64, POINTER(c_int64)]),
    "rr_static_param_bytes": (c_int, [POINTER(RrModel), POINTER(c_int64), POINTER(c_int64), POINTER(c_int64)]),
    "rr_cluster_validate": (c_int, [POINTER(RrCluster)]),
    "rr_validate_mesh": (c_int, [POINTER(RrMesh), POINTER(RrCluster)]),
    "rr_mesh_devices": (c_int, [POINTER(RrMesh), POINTER(RrCluster), POINTER(c_int32), c_int, POINTER(c_int)]),
    "rr_mesh_contains": (c_int, [POINTER(RrMesh), POINTER(RrCluster), c_int32, POINTER(c_int)]),
    "rr_enumerate_meshes": (c_int, [POINTER(RrCluster), POINTER(RrMesh), c_int, POINTER(c_int)]),
    "rr_overlap": (c_int, [POINTER(RrMesh), POINTER(RrMesh), POINTER(RrCluster), POINTER(c_int)]),
    "rr_link_bandwidth": (c_int, [POINTER(RrCluster), c_int32, c_int32, POINTER(c_double)]),
    "rr_mesh_to_string": (c_int, [POINTER(RrMesh), POINTER(RrCluster), POINTER(c_char), c_size_t, POINTER(c_size_t)]),
    "rr_mesh_from_string": (c_int, [c_char_p, POINTER(RrCluster), POINTER(RrMesh)]),
    "rr_stage_layer_map": (c_int, [c_int64, c_int, POINTER(c_int64), POINTER(c_int64)]),
    "rr_validate_placement": (c_int, [POINTER(RrModel), POINTER(RrPlacement), POINTER(RrCluster)]),
    "rr_plan_create": (c_int, [POINTER(RrModel), POINTER(RrPlacement), POINTER(RrPlacement), POINTER(RrCluster),
                               c_int, POINTER(_P)]),
    "rr_plan_destroy": (None, [_P]),
    "rr_plan_create_data": (c_int, [POINTER(RrPlacement), POINTER(RrPlacement), POINTER(RrCluster), c_int64, c_int,
                                    POINTER(_P)]),
    "rr_plan_totals": (c_int, [_P, POINTER(c_int64), POINTER(c_double)]),
    "rr_plan_num_ops": (c_int, [_P, c_int, POINTER(c_int)]),
    "rr_plan_get_op": (c_int, [_P, c_int, c_int, POINTER(RrOp)]),
    "rr_plan_to_json": (c_int, [_P, POINTER(c_char), c_size_t, POINTER(c_size_t)]),
    "rr_plan_shard_bytes": (c_int, [_P, c_int, c_int32, POINTER(c_int64)]),
    "rr_plan_device_traffic": (c_int, [_P, c_int32, POINTER(c_int64), POINTER(c_int64), POINTER(c_int64)]),
    "rr_plan_num_rects": (c_int, [_P, POINTER(c_int64)]),
    "rr_plan_layout": (c_int, [_P, c_int, c_int32, POINTER(c_int64), c_int64, POINTER(c_int64)]),
    "rr_plan_num_lowered": (c_int, [_P, POINTER(c_int)]),
    "rr_plan_get_lowered": (c_int, [_P, c_int, POINTER(c_int32), POINTER(c_int32), POINTER(c_int),
                                    POINTER(c_int64), c_int64, POINTER(c_int64)]),
    "rr_plan_work": (c_int, [_P, c_int, POINTER(c_int32), POINTER(c_int32), c_int, POINTER(c_int64)]),
    "rr_device_count": (c_int, [POINTER(c_int)]),
    "rr_device_alloc": (c_int, [c_int, c_size_t, POINTER(_P)]),
    "rr_device_free": (c_int, [_P]),
    "rr_host_alloc": (c_int, [c_size_t, POINTER(_P)]),
    "rr_host_free": (c_int, [_P]),
    "rr_memcpy": (c_int, [_P, _P, c_size_t, c_int, _P, c_int]),
    "rr_memset": (c_int, [_P, c_int, c_size_t, _P]),
    "rr_stream_sync": (c_int, [_P]),
    "rr_ipc_handle": (c_int, [_P, _P]),
    "rr_ipc_open": (c_int, [c_int, _P, POINTER(_P)]),
    "rr_ipc_close": (c_int, [_P]),
    "rr_enable_peer": (c_int, [c_int, c_int]),
    "rr_exec_create": (c_int, [_P, c_int, c_int, POINTER(_P), POINTER(_P), c_int, POINTER(c_int32),
                               POINTER(c_int32), c_int, c_int64, POINTER(_P)]),
    "rr_exec_launch": (c_int, [_P, _P, c_int]),
    "rr_exec_launch_fanout": (c_int, [_P, _P, c_int]),
    "rr_exec_enable_onload": (c_int, [_P, c_int, POINTER(c_int32), POINTER(c_int64), c_int64]),
    "rr_exec_launch_onload": (c_int, [_P, POINTER(_P), _P, _P, c_int]),
    "rr_exec_set_small_phase_bytes": (c_int, [_P, c_int64]),
    "rr_exec_launch_offload": (c_int, [_P, c_int, POINTER(c_int32), POINTER(c_int64), POINTER(_P), _P, _P]),
    "rr_exec_wire": (c_int, [_P, POINTER(c_int64), POINTER(c_int64)]),
    "rr_exec_set_kernel": (c_int, [_P, c_int]),
    "rr_exec_set_flag_kernel": (c_int, [_P, c_int]),
    "rr_exec_stats": (c_int, [_P, c_int, POINTER(c_int64), POINTER(c_int64), POINTER(c_int64)]),
    "rr_exec_destroy": (None, [_P]),
    "rr_fill_shard": (c_int, [_P, c_int, c_int32, _P, c_uint64, _P]),
    "rr_verify_shard": (c_int, [_P, c_int, c_int32, _P, c_uint64, _P, POINTER(c_int64), POINTER(c_int64)]),
    "rr_weight_value": (c_uint16, [c_uint64, c_int64, c_int64]),
    "rr_barrier_create": (c_int, [c_int, c_int, c_int, POINTER(_P), POINTER(_P)]),
    "rr_barrier_launch": (c_int, [_P, _P]),
    "rr_barrier_status": (c_int, [_P, POINTER(c_int)]),
    "rr_barrier_destroy": (None, [_P]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the CUDA extension has not been built "
            "(run `make -C paper_2406_14088_b200/csrc` or __graft_entry__.build()). "
            "There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class ValidationError(ValueError):
    """Mirror of rlplan::ValidationError (reference common.hpp:22-25)."""


class RrError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[rr status {status}] {message}")
        self.status = status


def check(status: int) -> None:
    if status == RR_OK:
        return
    msg = (lib.rr_last_error() or b"").decode()
    if status == RR_EINVAL:
        raise ValidationError(msg)
    raise RrError(status, msg)

