"""ctypes wrappers around ``sten_oracle.c`` plus a tiny pure-Python brute force.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Arrays are numpy: fp32 -> ``np.float32``; bf16 -> ``np.uint16`` bit patterns.
All functions return freshly allocated numpy arrays; nothing is cached.
"""
from __future__ import annotations

import ctypes
import itertools
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sten_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64 = ctypes.c_int64
_ptr = ctypes.c_void_p


def lib_path() -> str:
    return _LIB


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp.%d" % os.getpid()
        subprocess.check_call([
            "gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
            "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_sparsify.argtypes = [ctypes.c_int] * 4 + [_ptr, _i64, _i64, _i64, _ptr, _ptr]
        lib.oracle_densify.argtypes = [ctypes.c_int] * 4 + [_ptr, _ptr, _i64, _i64, _ptr, _i64]
        lib.oracle_spmm.argtypes = ([ctypes.c_int] * 4 + [_ptr, _ptr, _i64, _i64, _ptr, _i64, _i64,
                                                          _i64, _i64, _ptr, _ptr, ctypes.c_int])
        lib.oracle_dense_matmul.argtypes = [ctypes.c_int, _ptr, _i64, _i64, _i64, _ptr, _i64, _i64,
                                            _ptr, ctypes.c_int]
        lib.oracle_energy.argtypes = [ctypes.c_int, _ptr, _ptr, _i64, _i64, _i64]
        lib.oracle_same_format.argtypes = [ctypes.c_int] * 4 + [_ptr, _i64, _i64, _i64, _ptr, _ptr]
        lib.oracle_nmg_patterns.argtypes = [ctypes.c_int, ctypes.c_int, _ptr]
        lib.oracle_nmg_sparsify.argtypes = [ctypes.c_int] * 4 + [_ptr, _i64, _i64, _i64, _ptr, _ptr]
        lib.oracle_nmg_sparsify_exchange.argtypes = [ctypes.c_int] * 4 + [_ptr, _i64, _i64, _i64, ctypes.c_int,
                                                                          _ptr, _ptr]
        lib.oracle_sddmm.argtypes = [ctypes.c_int] * 4 + [_ptr, _i64, _i64, _ptr, _i64, _ptr, _ptr, _ptr, ctypes.c_int]
        lib.oracle_mask_check.argtypes = [ctypes.c_int] * 4 + [_ptr, _i64, _i64, _i64, _ptr, _ptr, _ptr]
        lib.oracle_nmg_densify.argtypes = [ctypes.c_int] * 4 + [_ptr, _ptr, _i64, _i64, _ptr, _i64]
        lib.oracle_nmg_spmm.argtypes = [ctypes.c_int] * 4 + [_ptr, _ptr, _i64, _i64, _ptr, _i64, _i64,
                                                             _ptr, _ptr, ctypes.c_int]
        lib.oracle_energy.restype = ctypes.c_double
        for f in (lib.oracle_sparsify, lib.oracle_densify, lib.oracle_spmm, lib.oracle_dense_matmul):
            f.restype = ctypes.c_int
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return 0
    if a.dtype == np.uint16:
        return 1
    raise TypeError("oracle arrays must be float32 or uint16 (bf16 bits), got %s" % a.dtype)


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError("%s failed with oracle status %d" % (what, rc))


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def sparsify(W: np.ndarray, n: int, m: int, g: int):
    """Return (values [M][K/m*n], idx [M/g][K/m][n] uint8) for a dense W [M][K]."""
    W = np.ascontiguousarray(W)
    M, K = W.shape
    dt = _dtype_code(W)
    if M % g or K % m:
        raise ValueError("shape (%d, %d) not divisible by g=%d / m=%d" % (M, K, g, m))
    values = np.zeros((M, K // m * n), dtype=W.dtype)
    idx = np.zeros((M // g, K // m, n), dtype=np.uint8)
    _check(_load().oracle_sparsify(n, m, g, dt, _p(W), M, K, K, _p(values), _p(idx)), "sparsify")
    return values, idx


def densify(values: np.ndarray, idx: np.ndarray, n: int, m: int, g: int, K: int) -> np.ndarray:
    values = np.ascontiguousarray(values)
    idx = np.ascontiguousarray(idx, dtype=np.uint8)
    M = values.shape[0]
    out = np.empty((M, K), dtype=values.dtype)
    _check(_load().oracle_densify(n, m, g, _dtype_code(values), _p(values), _p(idx), M, K,
                                  _p(out), K), "densify")
    return out


def spmm(values: np.ndarray, idx: np.ndarray, B: np.ndarray, n: int, m: int, g: int,
         cols: tuple | None = None, nthreads: int = 1, with_bound: bool = True):
    """fp64 reference C = mask(W) @ B (and Bound = |mask(W)| @ |B|).

    ``cols=(c0, c1)`` restricts the computation to a column slice; the
    returned arrays are then [M][c1-c0].
    """
    values = np.ascontiguousarray(values)
    idx = np.ascontiguousarray(idx, dtype=np.uint8)
    B = np.ascontiguousarray(B)
    if B.dtype != values.dtype:
        raise TypeError("values and B must share a dtype")
    M = values.shape[0]
    K, N = B.shape
    c0, c1 = (0, N) if cols is None else cols
    C = np.zeros((M, N), dtype=np.float64)
    Bd = np.zeros_like(C) if with_bound else None
    _check(_load().oracle_spmm(n, m, g, _dtype_code(values), _p(values), _p(idx), M, K, _p(B), N,
                               N, c0, c1, _p(C), _p(Bd) if with_bound else None, nthreads), "spmm")
    if cols is not None:
        C = C[:, c0:c1].copy()
        Bd = Bd[:, c0:c1].copy() if with_bound else None
    return (C, Bd) if with_bound else C


def dense_matmul(A: np.ndarray, B: np.ndarray, nthreads: int = 1) -> np.ndarray:
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B)
    M, K = A.shape
    K2, N = B.shape
    assert K == K2 and A.dtype == B.dtype
    C = np.empty((M, N), dtype=np.float64)
    _check(_load().oracle_dense_matmul(_dtype_code(A), _p(A), M, K, K, _p(B), N, N, _p(C), nthreads),
           "dense_matmul")
    return C


def energy(Xhat: np.ndarray, X: np.ndarray) -> float:
    """||X^||_1 / ||X||_1."""
    Xhat = np.ascontiguousarray(Xhat)
    X = np.ascontiguousarray(X)
    assert Xhat.shape == X.shape and Xhat.dtype == X.dtype
    M, K = X.shape
    return float(_load().oracle_energy(_dtype_code(X), _p(Xhat), _p(X), M, K, K))


def brute_select(W_int: np.ndarray, n: int, m: int, g: int) -> np.ndarray:
    """Exhaustive selection for tiny integer-valued W (pure Python).

    For every (group, m-block) enumerate all C(m, n) position subsets, sum the
    exact |w| of the group's rows over each subset in fp64 (exact for small
    integers), and keep the subset with the largest sum -- the argmax of the L1
    objective restricted to one group/block.  Ties go to the
    lexicographically smallest sorted subset.  Returns idx [M/g][K/m][n].
    """
    W = np.asarray(W_int, dtype=np.float64)
    M, K = W.shape
    G, KB = M // g, K // m
    out = np.zeros((G, KB, n), dtype=np.uint8)
    for grp in range(G):
        rows = W[grp * g:(grp + 1) * g]
        for kb in range(KB):
            blk = np.abs(rows[:, kb * m:(kb + 1) * m])
            best, best_sum = None, -1.0
            for subset in itertools.combinations(range(m), n):  # lexicographic order
                tot = float(sum(blk[i][j] for i in range(g) for j in subset))
                if tot > best_sum:
                    best, best_sum = subset, tot
            out[grp, kb] = best
    return out


# ---------------------------------------------------------------------------------------------
# Chunked n:m:g -- the paper's own format (R17-R21)
# ---------------------------------------------------------------------------------------------
def nmg_patterns(n: int, m: int) -> np.ndarray:
    """The C(m,n) patterns in the fixed (revolving-door) order: [C][n] ascending positions."""
    C = comb(m, n)
    pos = np.zeros((C, n), dtype=np.int32)
    _check(_load().oracle_nmg_patterns(n, m, _p(pos)), "nmg_patterns")
    return pos


def comb(m: int, n: int) -> int:
    import math
    return math.comb(m, n)


def nmg_chunk(n: int, m: int, g: int) -> int:
    """L = C(m,n) * g columns per chunk."""
    return comb(m, n) * g


def nmg_sparsify(W: np.ndarray, n: int, m: int, g: int):
    """Greedy conversion to chunked n:m:g: (values [M/m][K/L][L][n], idx [M/m][K/L][L] uint16)."""
    W = np.ascontiguousarray(W)
    M, K = W.shape
    L = nmg_chunk(n, m, g)
    if M % m or K % L:
        raise ValueError("shape (%d, %d) not divisible by m=%d / L=%d" % (M, K, m, L))
    values = np.zeros((M // m, K // L, L, n), dtype=W.dtype)
    idx = np.zeros((M // m, K // L, L), dtype=np.uint16)
    _check(_load().oracle_nmg_sparsify(n, m, g, _dtype_code(W), _p(W), M, K, K, _p(values), _p(idx)),
           "nmg_sparsify")
    return values, idx


def nmg_sparsify_exchange(W: np.ndarray, n: int, m: int, g: int, init: int = 0):
    """The paper's GPU conversion, sequential reading DESIGN.md R22: pairwise
    pattern swaps that raise the pair's magnitude until a pass makes none.  init 0 = column b starts
    with pattern b / g, 1 = start from the greedy.  Same layout as nmg_sparsify."""
    W = np.ascontiguousarray(W)
    M, K = W.shape
    L = nmg_chunk(n, m, g)
    if M % m or K % L:
        raise ValueError("shape (%d, %d) not divisible by m=%d / L=%d" % (M, K, m, L))
    values = np.zeros((M // m, K // L, L, n), dtype=W.dtype)
    idx = np.zeros((M // m, K // L, L), dtype=np.uint16)
    _check(_load().oracle_nmg_sparsify_exchange(n, m, g, _dtype_code(W), _p(W), M, K, K, int(init), _p(values),
                                                _p(idx)), "nmg_sparsify_exchange")
    return values, idx


def nmg_densify(values: np.ndarray, idx: np.ndarray, n: int, m: int, g: int, K: int) -> np.ndarray:
    values = np.ascontiguousarray(values)
    idx = np.ascontiguousarray(idx, dtype=np.uint16)
    M = values.shape[0] * m
    out = np.empty((M, K), dtype=values.dtype)
    _check(_load().oracle_nmg_densify(n, m, g, _dtype_code(values), _p(values), _p(idx), M, K, _p(out), K),
           "nmg_densify")
    return out


def nmg_spmm(values: np.ndarray, idx: np.ndarray, B: np.ndarray, n: int, m: int, g: int, nthreads: int = 1):
    """fp64 C = mask(W) @ B for chunked n:m:g, and Bound = |mask(W)| @ |B|."""
    values = np.ascontiguousarray(values)
    idx = np.ascontiguousarray(idx, dtype=np.uint16)
    B = np.ascontiguousarray(B)
    if B.dtype != values.dtype:
        raise TypeError("values and B must share a dtype")
    M = values.shape[0] * m
    K, N = B.shape
    C = np.zeros((M, N), dtype=np.float64)
    Bd = np.zeros_like(C)
    _check(_load().oracle_nmg_spmm(n, m, g, _dtype_code(values), _p(values), _p(idx), M, K, _p(B), N, N,
                                   _p(C), _p(Bd), nthreads), "nmg_spmm")
    return C, Bd


def nmg_brute_best_energy(W_int: np.ndarray, n: int, m: int, g: int) -> float:
    """Exhaustive optimum of the L1 objective over every valid chunked
    n:m:g mask of a tiny integer W (one row block, one chunk): every assignment of the L
    columns to patterns with each pattern used exactly g times.  Returns the kept L1 mass."""
    W = np.abs(np.asarray(W_int, dtype=np.float64))
    M, K = W.shape
    L = nmg_chunk(n, m, g)
    assert M == m and K == L
    pats = list(itertools.combinations(range(m), n))
    best = -1.0

    def rec(b, cnt, tot):
        nonlocal best
        if b == L:
            best = max(best, tot)
            return
        for p, P in enumerate(pats):
            if cnt[p] < g:
                cnt[p] += 1
                rec(b + 1, cnt, tot + sum(W[i, b] for i in P))
                cnt[p] -= 1

    rec(0, [0] * len(pats), 0.0)
    return best


def same_format(W: np.ndarray, idx: np.ndarray, n: int, m: int, g: int) -> np.ndarray:
    """SameFormat re-sparsification: values of W at an existing pattern idx."""
    W = np.ascontiguousarray(W)
    idx = np.ascontiguousarray(idx, dtype=np.uint8)
    M, K = W.shape
    values = np.zeros((M, K // m * n), dtype=W.dtype)
    _check(_load().oracle_same_format(n, m, g, _dtype_code(W), _p(W), M, K, K, _p(idx), _p(values)),
           "same_format")
    return values


def sddmm(G: np.ndarray, B: np.ndarray, idx: np.ndarray, n: int, m: int, g: int, nthreads: int = 1):
    """Weight gradient of C = densify(values, idx) @ B in the values layout (NEXT-2 masked linear):
    dV[r][kb n + t] = sum_c G[r][c] B[kb m + idx[r/g][kb][t]][c] in fp64, and Bound = sum |G||B|."""
    G = np.ascontiguousarray(G)
    B = np.ascontiguousarray(B)
    idx = np.ascontiguousarray(idx, dtype=np.uint8)
    M, N = G.shape
    K = B.shape[0]
    assert B.shape[1] == N and G.dtype == B.dtype
    dV = np.zeros((M, K // m * n), np.float64)
    bound = np.zeros_like(dV)
    _check(_load().oracle_sddmm(n, m, g, _dtype_code(G), _p(G), M, N, _p(B), K, _p(idx), _p(dV), _p(bound),
                                int(nthreads)), "sddmm")
    return dV, bound


def mask_check(W: np.ndarray, idx: np.ndarray, n: int, m: int, g: int):
    """Fixed-mask fast path: (SameFormat values of W at idx, #nonzeros of W outside
    the pattern)."""
    W = np.ascontiguousarray(W)
    idx = np.ascontiguousarray(idx, dtype=np.uint8)
    M, K = W.shape
    values = np.zeros((M, K // m * n), dtype=W.dtype)
    out = np.zeros(1, np.int64)
    _check(_load().oracle_mask_check(n, m, g, _dtype_code(W), _p(W), M, K, K, _p(idx), _p(values), _p(out)),
           "mask_check")
    return values, int(out[0])


# ---------------------------------------------------------------------------------------------
# NEXT-3 epilogue (bias + activation of a BERT linear), fp64
# ---------------------------------------------------------------------------------------------
def gelu(x: np.ndarray) -> np.ndarray:
    """GELU, erf form: x/2 (1 + erf(x / sqrt 2)) in fp64 (math.erf per element; small inputs)."""
    import math
    f = np.frompyfunc(lambda t: 0.5 * t * (1.0 + math.erf(t / math.sqrt(2.0))), 1, 1)
    return f(np.asarray(x, dtype=np.float64)).astype(np.float64)


def bias_act(C: np.ndarray, bias: np.ndarray | None, act: int) -> np.ndarray:
    """act(C + bias[:, None]) in fp64; act 0 none, 1 GELU, 2 ReLU."""
    y = np.asarray(C, dtype=np.float64)
    if bias is not None:
        y = y + np.asarray(bias, dtype=np.float64)[:, None]
    if act == 1:
        y = gelu(y)
    elif act == 2:
        y = np.maximum(y, 0.0)
    return y
