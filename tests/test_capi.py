"""The drop-in boundary: librrealloc.so loads without a GPU, exports every
entry point include/rr_realloc.h declares, and reports errors the way the
reference does (ValidationError text through rr_last_error)."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

from paper_2406_14088_b200 import _lib
from paper_2406_14088_b200 import rlplan as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rr_realloc.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rr_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_bound_symbols():
    assert declared_symbols() == sorted(_lib.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_no_torch_or_cuda_types_in_signatures():
    text = open(HEADER).read()
    assert "torch" not in re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    assert "cudaStream_t" not in re.sub(r"/\*.*?\*/", "", text, flags=re.S)


def test_abi_version_and_error_reporting():
    assert _lib.lib.rr_abi_version() == 5
    bad = P.ModelSpec(name="x", hidden_size=100, intermediate_size=8, num_layers=1, num_attention_heads=3,
                      num_kv_heads=1, vocab_size=10, max_position_embeddings=16)
    with pytest.raises(P.ValidationError, match="ModelSpec 'x': hidden_size must be divisible by num_attention_heads"):
        P.param_count(bad, True)
    st = _lib.lib.rr_param_count(ctypes.byref(bad._c()), 1, ctypes.byref(ctypes.c_int64()))
    assert st == _lib.RR_EINVAL
    assert b"divisible" in _lib.lib.rr_last_error()


def test_buffer_too_small_reports_needed_size():
    c = P.b200_cluster(8)
    m = P.DeviceMesh(0, 1, 0, 4)
    buf = ctypes.create_string_buffer(4)
    need = ctypes.c_size_t()
    st = _lib.lib.rr_mesh_to_string(ctypes.byref(m._c()), ctypes.byref(c._c()), buf, 4, ctypes.byref(need))
    assert st == _lib.RR_ERANGE and need.value == len("trainer01:gpu[0-3]") + 1


def test_device_calls_fail_loudly_without_gpu():
    """No CPU fallback: with no CUDA device the execution entry points error out."""
    from paper_2406_14088_b200 import runtime as R
    if R.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(_lib.RrError):
        R.DeviceBuffer(0, 1024)
