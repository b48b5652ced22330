"""CPU-side checks of the C-ABI boundary: the library builds, loads, and exports
every entry point include/stan_cl.h declares (no compute calls: no GPU here)."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stan_cl.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(stan_cl_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_1907_01063_b200 import _build
    return _build.build()


def test_header_declares_boundary():
    syms = declared_symbols()
    for need in ("stan_cl_cholesky", "stan_cl_cholesky_adjoint", "stan_cl_gp_exp_quad_cov"):
        assert need in syms


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (stan_cl_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_binding_signatures_cover_header(lib_path):
    import paper_1907_01063_b200 as sc
    assert set(sc.SIGNATURES) == set(declared_symbols())
    lib = sc.load()
    assert lib.stan_cl_version() >= 100
    # pure host-side calls (no device work)
    assert lib.stan_cl_status_string(-1) == b"invalid argument"
    assert lib.stan_cl_set_block_size(256) == 0 and lib.stan_cl_get_block_size() == 256
    assert lib.stan_cl_set_block_size(0) == 0 and lib.stan_cl_get_block_size() == 0
    assert lib.stan_cl_set_block_size(96) == -1
    assert lib.stan_cl_workspace_bytes(0) == 256         # the status header alone
    assert lib.stan_cl_workspace_bytes(16384) > 16384 * 128 * 8


def test_sm100a_code_in_library(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib_path], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass                       # FP64 tensor-core path present
    assert "LDGSTS" in sass                           # cp.async staging


def test_no_oracle_in_product_path():
    # the product package must not import or link the oracle
    pkg = os.path.join(ROOT, "paper_1907_01063_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt and "oracle.c" not in txt, f
