"""C++ drop-in: a reference-style rlplan caller compiles against include/
and links librrealloc.so; the model-arith/cluster subset also compiles
against the reference's own headers (ABI-compatible declarations)."""
from __future__ import annotations

import os
import subprocess

import pytest

from paper_2406_14088_b200._lib import LIB_PATH

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_main.cpp")
REF_INCLUDE = "/root/reference/proj/include"


def _build_and_run(tmp_path, include, defines=()):
    exe = str(tmp_path / "dropin")
    cmd = ["g++", "-std=c++20", "-O1", f"-I{include}", *defines, SRC, LIB_PATH,
           f"-Wl,-rpath,{os.path.dirname(LIB_PATH)}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return subprocess.run([exe], check=True, capture_output=True, text=True).stdout


def test_cpp_caller_against_product_headers(tmp_path):
    out = _build_and_run(tmp_path, os.path.join(ROOT, "include"))
    assert "param_count 8030261248 7504924672" in out
    assert "meshes 15" in out
    assert "mesh trainer01:gpu[4-7] first 4" in out
    assert "error DeviceMesh: sub-node mesh offset must be aligned to its size" in out
    assert "plan ops 8 local 16 total 112419930112" in out
    assert "stages [0,3) [3,5)" in out


@pytest.mark.skipif(not os.path.isdir(REF_INCLUDE), reason="reference headers not mounted")
def test_cpp_caller_against_reference_headers(tmp_path):
    out = _build_and_run(tmp_path, REF_INCLUDE, ["-DREF_HEADERS_ONLY"])
    assert "param_count 8030261248 7504924672" in out
    assert "mesh trainer01:gpu[4-7] first 4" in out
    assert "error DeviceMesh: sub-node mesh offset must be aligned to its size" in out
