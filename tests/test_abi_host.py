"""Host-side checks of the C ABI (-m "not gpu"): the library builds for sm_100a,
loads, exports every symbol include/sten.h declares, and its argument
validation / planning logic behaves as documented -- without any kernel launch.
"""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2304_07613_b200 as pkg
from paper_2304_07613_b200 import sten

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sten.h")

OK, INVALID, SHAPE, UNSUPPORTED = 0, 1, 2, 3


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sten_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(sten.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = sten.load()
    out = subprocess.check_output(["nm", "-D", "--defined-only", sten.lib_path()]).decode()
    exported = set(re.findall(r"\bT (sten_[a-z0-9_]+)", out))
    for name in declared_functions():
        assert name in exported, name
        assert getattr(lib, name) is not None


def test_library_is_sm100a():
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sten.lib_path()]).decode()
    assert "sm_100a" in out


def test_status_and_names():
    assert sten.status_string(0) == "STEN_OK"
    assert sten.status_string(3) == "STEN_ERR_UNSUPPORTED"
    assert sten.algo_name(1) == "simt" and sten.algo_name(2) == "mma_sync"
    assert sten.load().sten_version() >= 1


FAKE = 1 << 20   # a non-null, 16-byte aligned dummy address; never dereferenced on error paths


def _sparsify(n, m, g, dt, W, M, K, ldw, V=FAKE, I=FAKE):
    return sten.load().sten_sparsify_grouped_nm(sten.sten_nmg(n, m, g), dt, W, M, K, ldw, V, I, None)


def _spmm(n, m, g, dt, M, K, ldb, N, ldc, B=FAKE, C=FAKE, cdt=None, plan=None):
    lib = sten.load()
    args = (sten.sten_nmg(n, m, g), dt, FAKE, FAKE, M, K, B, ldb, N, C, ldc, dt if cdt is None else cdt)
    if plan is None:
        return lib.sten_spmm_grouped_nm(*args, None)
    return lib.sten_spmm_grouped_nm_ex(*args, ctypes.byref(plan), None)


@pytest.mark.parametrize("n,m,g,expect", [
    (0, 4, 4, INVALID), (4, 4, 4, INVALID), (2, 4, 0, INVALID), (1, 17, 1, INVALID),
    (2, 5, 1, UNSUPPORTED), (2, 14, 1, UNSUPPORTED),
])
def test_format_validation(n, m, g, expect):
    assert _sparsify(n, m, g, 0, FAKE, 64, 64, 64) == expect


def test_shape_and_pointer_validation():
    assert _sparsify(2, 4, 4, 0, None, 64, 64, 64) == INVALID          # null W
    assert _sparsify(2, 4, 4, 0, FAKE, 62, 64, 64) == SHAPE            # M % g
    assert _sparsify(2, 4, 4, 0, FAKE, 64, 66, 66) == SHAPE            # K % m
    assert _sparsify(2, 4, 4, 0, FAKE, 64, 64, 60) == SHAPE            # ldw < K
    assert _sparsify(2, 4, 4, 7, FAKE, 64, 64, 64) == INVALID          # dtype
    assert _spmm(2, 4, 4, 0, 64, 64, 30, 32, 32) == SHAPE              # ldb < N
    assert _spmm(2, 4, 4, 0, 64, 64, 32, 32, 16) == SHAPE              # ldc < N
    assert _spmm(2, 4, 4, 0, 64, 64, 33, 33, 33) == UNSUPPORTED        # fp32 ldb % 4
    assert _spmm(2, 4, 4, 1, 64, 64, 36, 36, 36) == UNSUPPORTED        # bf16 ldb % 8
    assert _spmm(2, 4, 4, 0, 64, 64, 32, 32, 32, B=FAKE + 4) == UNSUPPORTED   # misaligned B
    assert _spmm(2, 4, 4, 0, 64, 64, 32, 32, 32, B=None) == INVALID


def test_plan_override_validation():
    bad_tile = sten.make_plan(algo=sten.ALGO_SIMT, tile=9)
    assert _spmm(2, 4, 4, 0, 64, 64, 32, 32, 32, plan=bad_tile) == UNSUPPORTED
    mma_f32 = sten.make_plan(algo=sten.ALGO_MMA_SYNC)
    assert _spmm(2, 4, 8, 0, 64, 64, 32, 32, 32, plan=mma_f32) == UNSUPPORTED   # mma needs bf16
    mma_g4 = sten.make_plan(algo=sten.ALGO_MMA_SYNC)
    assert _spmm(2, 4, 4, 1, 64, 64, 32, 32, 32, plan=mma_g4) == UNSUPPORTED    # mma needs 8 | g


def test_empty_problems_are_noops():
    # M == 0 / N == 0 return OK before touching the device
    assert _spmm(2, 4, 4, 0, 0, 64, 32, 32, 32) == OK
    assert _spmm(2, 4, 4, 0, 64, 64, 0, 0, 0) == OK
    assert _sparsify(2, 4, 4, 0, FAKE, 0, 64, 64) == OK


def test_plan_query():
    p = sten.spmm_plan(2, 4, 4, 768, 3072, 1024)
    assert p.algo == sten.ALGO_SIMT and 1 <= p.split_k <= 16 and p.tile >= 1
    bf16 = __import__("torch").bfloat16
    # bf16, 16 | g, at least one full wave of 256 x 128 tiles: tcgen05 with the largest RB | g
    p = sten.spmm_plan(2, 4, 16, 1024, 4096, 16384, ab_dtype=bf16)
    assert p.algo == sten.ALGO_TCGEN05 and p.tile == 1 and p.split_k == 1
    assert sten.spmm_plan(1, 4, 64, 1024, 4096, 16384, ab_dtype=bf16).tile == 3
    # small grids keep the split-K mma.sync path
    p = sten.spmm_plan(2, 4, 16, 768, 768, 1024, ab_dtype=bf16)
    assert p.algo == sten.ALGO_MMA_SYNC
    # the plan is a pure function of the shape
    assert sten.spmm_plan(1, 4, 4, 768, 768, 1024).as_dict() == sten.spmm_plan(1, 4, 4, 768, 768, 1024).as_dict()


def test_workspace_size():
    ws = sten.sparse_linear_host_workspace_size(2, 4, 4, 64, 64, 32)
    assert ws >= 64 * 64 * 4 + 64 * 32 * 4 + 64 * 32 * 4 + 64 * 32 * 4
    assert sten.sparse_linear_host_workspace_size(2, 4, 4, 62, 64, 32) == -1


def test_package_has_no_oracle_dependency():
    src_dir = os.path.dirname(pkg.__file__)
    for root, _, files in os.walk(src_dir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(root, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "sten_oracle" not in text, f
