"""Thin ctypes binding of the C ABI in include/sten.h (argument marshalling only).

Every function forwards torch CUDA tensors' device pointers and the current
CUDA stream to ``libsten.so``; all computation happens in the library's
sm_100a kernels.  There is no CPU fallback: if the library or a CUDA device is
missing, the calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os

import torch

from . import build as _build

F32, BF16 = 0, 1
ALGO_AUTO, ALGO_SIMT, ALGO_MMA_SYNC, ALGO_TCGEN05 = 0, 1, 2, 3
_STATUS = {0: "STEN_OK", 1: "STEN_ERR_INVALID_ARG", 2: "STEN_ERR_SHAPE",
           3: "STEN_ERR_UNSUPPORTED", 4: "STEN_ERR_CUDA"}


class StenError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__("%s failed: %s" % (what, _STATUS.get(status, status)))
        self.status = status


class sten_nmg(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("m", ctypes.c_int32), ("g", ctypes.c_int32)]


class sten_spmm_problem(ctypes.Structure):
    _fields_ = [("f", sten_nmg), ("reserved", ctypes.c_int32), ("values", ctypes.c_void_p), ("idx", ctypes.c_void_p),
                ("M", ctypes.c_int64), ("K", ctypes.c_int64), ("B", ctypes.c_void_p), ("ldb", ctypes.c_int64),
                ("N", ctypes.c_int64), ("C", ctypes.c_void_p), ("ldc", ctypes.c_int64)]


class sten_sparsify_problem(ctypes.Structure):
    _fields_ = [("f", sten_nmg), ("reserved", ctypes.c_int32), ("W", ctypes.c_void_p), ("M", ctypes.c_int64),
                ("K", ctypes.c_int64), ("ldw", ctypes.c_int64), ("values", ctypes.c_void_p), ("idx", ctypes.c_void_p)]


class sten_host_linear_problem(ctypes.Structure):
    _fields_ = [("f", sten_nmg), ("reserved", ctypes.c_int32), ("W_host", ctypes.c_void_p), ("M", ctypes.c_int64),
                ("K", ctypes.c_int64), ("ldw", ctypes.c_int64), ("B_host", ctypes.c_void_p), ("ldb", ctypes.c_int64),
                ("N", ctypes.c_int64), ("C_host", ctypes.c_void_p), ("ldc", ctypes.c_int64),
                ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_int64)]


class sten_spmm_plan(ctypes.Structure):
    _fields_ = [("algo", ctypes.c_int32), ("split_k", ctypes.c_int32), ("tile", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 5)]

    def as_dict(self):
        return {"algo": self.algo, "split_k": self.split_k, "tile": self.tile}


_lib = None
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p

# exported symbols and their ctypes signatures (kept in sync with include/sten.h)
SIGNATURES = {
    "sten_sparsify_grouped_nm": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "sten_densify": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "sten_spmm_grouped_nm": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _vp, _i64, _i64, _vp, _i64, _i64,
                                            _vp, _i64, ctypes.c_int, _vp]),
    "sten_spmm_plan_query": (ctypes.c_int, [sten_nmg, ctypes.c_int, _i64, _i64, _i64, ctypes.c_int,
                                            ctypes.POINTER(sten_spmm_plan)]),
    "sten_spmm_grouped_nm_ex": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _vp, _i64, _i64, _vp, _i64, _i64,
                                               _vp, _i64, ctypes.c_int, ctypes.POINTER(sten_spmm_plan), _vp]),
    "sten_spmm_autotune": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _vp, _i64, _i64, _vp, _i64, _i64,
                                          _vp, _i64, ctypes.c_int, ctypes.c_int32, _vp,
                                          ctypes.POINTER(sten_spmm_plan)]),
    "sten_sparse_linear_host_workspace_size": (ctypes.c_int64, [sten_nmg, ctypes.c_int, _i64, _i64, _i64,
                                                                ctypes.c_int]),
    "sten_sparse_linear_host": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _i64, _i64, _i64, _vp, _i64, _i64,
                                               _vp, _i64, ctypes.c_int, _vp, _i64, _vp]),
    "sten_nmg_sparsify": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "sten_nmg_sparsify_ex": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _i64, _i64, _i64, _vp, _vp,
                                            ctypes.c_int32, _vp]),
    "sten_nmg_densify": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "sten_nmg_spmm": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _vp, _i64, _i64, _vp, _i64, _i64,
                                     _vp, _i64, ctypes.c_int, _vp]),
    "sten_sparse_linear_host_async": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _i64, _i64, _i64, _vp, _i64,
                                                     _i64, _vp, _i64, ctypes.c_int, _vp, _i64, _vp]),
    "sten_sparse_linear_host_pipelined_async": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(sten_host_linear_problem),
                                                               ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]),
    "sten_resparsify_same_format": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _i64, _i64, _i64, _vp, _vp,
                                                   _vp]),
    "sten_spmm_grouped_nm_allgather": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _vp, _i64, _i64, _vp, _i64,
                                                      _i64, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32,
                                                      _i64, _i64, ctypes.c_int, ctypes.POINTER(sten_spmm_plan),
                                                      _vp]),
    "sten_spmm_grouped_nm_bias_act": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _vp, _i64, _i64, _vp, _i64,
                                                     _i64, _vp, _i64, ctypes.c_int, _vp, ctypes.c_int32,
                                                     ctypes.POINTER(sten_spmm_plan), _vp]),
    "sten_spmm_grouped_nm_batched": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(sten_spmm_problem),
                                                    ctypes.c_int32, _vp]),
    "sten_spmm_grouped_nm_batched_ex": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(sten_spmm_problem),
                                                       ctypes.POINTER(ctypes.c_int32), ctypes.c_int32, _vp, _i64,
                                                       _vp]),
    "sten_spmm_batched_workspace_size": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(sten_spmm_problem),
                                                        ctypes.POINTER(ctypes.c_int32), ctypes.c_int32,
                                                        ctypes.POINTER(_i64)]),
    "sten_sparsify_grouped_nm_batched": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(sten_sparsify_problem),
                                                        ctypes.c_int, _vp]),
    "sten_mask_check_repack": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _i64, _i64, _i64, _vp, _vp, _vp,
                                              _vp]),
    "sten_sddmm_grouped_nm": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _i64, _i64, _i64, _vp, _i64, _i64,
                                             _vp, _vp, ctypes.c_int, _vp]),
    "sten_spmm_grouped_nm_epilogue": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _vp, _i64, _i64, _vp, _i64,
                                                     _i64, _vp, _i64, ctypes.c_int, _vp, ctypes.c_int32, _vp, _i64,
                                                     ctypes.POINTER(sten_spmm_plan), _vp]),
    "sten_sp24_packed_size": (ctypes.c_int, [sten_nmg, _i64, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "sten_sp24_pack": (ctypes.c_int, [sten_nmg, ctypes.c_int, _vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "sten_spmm_sp24": (ctypes.c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _i64, _vp, _i64, ctypes.c_int,
                                      ctypes.c_int32, _vp]),
    "sten_spmm_sp24_epilogue": (ctypes.c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _i64, _vp, _i64, ctypes.c_int,
                                               _vp, ctypes.c_int32, _vp, _i64, ctypes.c_int32, _vp]),
    "sten_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "sten_algo_name": (ctypes.c_char_p, [ctypes.c_int32]),
    "sten_spmm_launch_count": (ctypes.c_int32, [ctypes.POINTER(sten_spmm_plan)]),
    "sten_version": (ctypes.c_int32, []),
}


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libsten.so (building it in-tree first if it is missing or stale)."""
    global _lib
    if _lib is None:
        if build_if_missing and _build.needs_build():
            _build.build()
        if not os.path.exists(_build.LIB):
            raise RuntimeError("libsten.so is missing (run paper_2304_07613_b200/build.py); "
                               "there is no CPU fallback")
        # STEN_LIB_PATH: load an instrumented debug build instead (tools/phase_timing.py)
        lib = ctypes.CDLL(os.environ.get("STEN_LIB_PATH", _build.LIB))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.bfloat16:
        return BF16
    raise TypeError("sten supports float32 and bfloat16 tensors, got %s" % t.dtype)


def _torch_dtype(code: int):
    return torch.float32 if code == F32 else torch.bfloat16


def _cuda(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError("%s must be a CUDA tensor (no CPU fallback)" % name)
    if t.dim() != 2 and name not in ("idx",):
        raise ValueError("%s must be 2-D" % name)


def _check_operands(values: torch.Tensor, idx: torch.Tensor, B: torch.Tensor):
    """The C ABI assumes packed values [M][K'] / idx [M/g][K/m][n] on the current device and one
    A/B element type: reject anything else instead of letting the kernel reinterpret bytes."""
    _cuda(values, "values")
    _cuda(B, "B")
    if values.dtype != B.dtype:
        raise TypeError("values (%s) and B (%s) must share a dtype" % (values.dtype, B.dtype))
    if idx.dtype != torch.uint8:
        raise TypeError("idx must be uint8")
    if not values.is_contiguous() or not idx.is_contiguous():
        raise ValueError("values and idx must be contiguous (packed [M][K'] / [M/g][K/m][n])")
    dev = torch.cuda.current_device()
    for t, nm in ((values, "values"), (idx, "idx"), (B, "B")):
        if t.device.index != dev:
            raise ValueError("%s is on cuda:%s, the current device is cuda:%d" % (nm, t.device.index, dev))


def _ld(t: torch.Tensor) -> int:
    if t.stride(-1) != 1:
        raise ValueError("innermost dimension must be contiguous")
    return t.stride(0) if t.dim() == 2 else t.shape[-1]


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _check(status: int, what: str):
    if status != 0:
        raise StenError(status, what)


def sparsify_grouped_nm(W: torch.Tensor, n: int, m: int, g: int, values: torch.Tensor | None = None,
                        idx: torch.Tensor | None = None, stream=None):
    """a1-a3: dense W [M][K] -> (values [M][K/m*n], idx [M/g][K/m][n] uint8)."""
    _cuda(W, "W")
    M, K = W.shape
    if values is None:
        values = torch.empty((M, K // m * n if m else 0), dtype=W.dtype, device=W.device)
    if idx is None:
        idx = torch.empty((M // g if g else 0, K // m if m else 0, n), dtype=torch.uint8, device=W.device)
    _check(load().sten_sparsify_grouped_nm(sten_nmg(n, m, g), _dt(W), W.data_ptr(), M, K, _ld(W),
                                           values.data_ptr(), idx.data_ptr(), _stream(stream)),
           "sten_sparsify_grouped_nm")
    return values, idx


def sparsify_grouped_nm_batched(problems, stream=None):
    """a1-a3 for several weights in as few launches as possible: problems = [(W, n, m, g, values, idx), ...]
    (sten_sparsify_grouped_nm_batched; same bits as one sparsify_grouped_nm per weight)."""
    arr = (sten_sparsify_problem * len(problems))()
    dt = None
    for k, (W, n, m, g, values, idx) in enumerate(problems):
        _cuda(W, "W")
        if dt is None:
            dt = W.dtype
        if W.dtype != dt or values.dtype != dt or idx.dtype != torch.uint8:
            raise TypeError("one dtype for every W / values, uint8 idx")
        if not values.is_contiguous() or not idx.is_contiguous():
            raise ValueError("values and idx must be contiguous")
        arr[k].f = sten_nmg(n, m, g)
        arr[k].W, arr[k].M, arr[k].K, arr[k].ldw = W.data_ptr(), W.shape[0], W.shape[1], _ld(W)
        arr[k].values, arr[k].idx = values.data_ptr(), idx.data_ptr()
    _check(load().sten_sparsify_grouped_nm_batched(len(problems), arr, _dt(problems[0][0]), _stream(stream)),
           "sten_sparsify_grouped_nm_batched")
    return [(p[4], p[5]) for p in problems]


def resparsify_same_format(W: torch.Tensor, idx: torch.Tensor, n: int, m: int, g: int,
                           values: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """NEXT-2 SameFormat: values of a new dense W [M][K] at the existing pattern idx."""
    _cuda(W, "W")
    M, K = W.shape
    if values is None:
        values = torch.empty((M, K // m * n), dtype=W.dtype, device=W.device)
    _check(load().sten_resparsify_same_format(sten_nmg(n, m, g), _dt(W), W.data_ptr(), M, K, _ld(W),
                                              idx.data_ptr(), values.data_ptr(), _stream(stream)),
           "sten_resparsify_same_format")
    return values


def mask_check_repack(W: torch.Tensor, idx: torch.Tensor, n: int, m: int, g: int,
                      values: torch.Tensor | None = None, stream=None):
    """Fixed-mask fast path: (SameFormat values of W at idx, device int64 tensor = #nonzeros of W outside
    the pattern) in one pass (sten_mask_check_repack)."""
    _cuda(W, "W")
    M, K = W.shape
    if values is None:
        values = torch.empty((M, K // m * n), dtype=W.dtype, device=W.device)
    outside = torch.empty((1,), dtype=torch.int64, device=W.device)
    _check(load().sten_mask_check_repack(sten_nmg(n, m, g), _dt(W), W.data_ptr(), M, K, _ld(W), idx.data_ptr(),
                                         values.data_ptr(), outside.data_ptr(), _stream(stream)),
           "sten_mask_check_repack")
    return values, outside


def sddmm_grouped_nm(G: torch.Tensor, B: torch.Tensor, idx: torch.Tensor, n: int, m: int, g: int,
                     out: torch.Tensor | None = None, out_dtype=None, stream=None) -> torch.Tensor:
    """dV [M][K/m*n] = (G @ B^T) sampled at the kept positions (the masked linear's weight gradient in the
    values layout; sten_sddmm_grouped_nm).  G [M][N], B [K][N]."""
    _cuda(G, "G")
    _cuda(B, "B")
    if G.dtype != B.dtype:
        raise TypeError("G and B must share a dtype")
    M, N = G.shape
    K = B.shape[0]
    if out is None:
        out = torch.empty((M, K // m * n), dtype=out_dtype or G.dtype, device=G.device)
    _check(load().sten_sddmm_grouped_nm(sten_nmg(n, m, g), _dt(G), G.data_ptr(), M, N, _ld(G), B.data_ptr(), K,
                                        _ld(B), idx.data_ptr(), out.data_ptr(), _dt(out), _stream(stream)),
           "sten_sddmm_grouped_nm")
    return out


def densify(values: torch.Tensor, idx: torch.Tensor, n: int, m: int, g: int, K: int,
            out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """a4: grouped n:m -> dense [M][K] (zeros at pruned positions)."""
    _cuda(values, "values")
    M = values.shape[0]
    if out is None:
        out = torch.empty((M, K), dtype=values.dtype, device=values.device)
    _check(load().sten_densify(sten_nmg(n, m, g), _dt(values), values.data_ptr(), idx.data_ptr(), M, K,
                               out.data_ptr(), _ld(out), _stream(stream)), "sten_densify")
    return out


def spmm_plan(n: int, m: int, g: int, M: int, K: int, N: int, ab_dtype=torch.float32,
              c_dtype=None) -> sten_spmm_plan:
    plan = sten_spmm_plan()
    ab = F32 if ab_dtype == torch.float32 else BF16
    c = ab if c_dtype is None else (F32 if c_dtype == torch.float32 else BF16)
    _check(load().sten_spmm_plan_query(sten_nmg(n, m, g), ab, M, K, N, c, ctypes.byref(plan)),
           "sten_spmm_plan_query")
    return plan


def make_plan(algo: int = ALGO_AUTO, split_k: int = 0, tile: int = 0) -> sten_spmm_plan:
    p = sten_spmm_plan()
    p.algo, p.split_k, p.tile = algo, split_k, tile
    return p


def spmm_grouped_nm(values: torch.Tensor, idx: torch.Tensor, B: torch.Tensor, n: int, m: int, g: int,
                    out: torch.Tensor | None = None, out_dtype=None, plan: sten_spmm_plan | None = None,
                    stream=None) -> torch.Tensor:
    """a5-a7: C [M][N] = densify(values, idx) @ B  (B [K][N])."""
    _check_operands(values, idx, B)
    M = values.shape[0]
    K, N = B.shape
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype or B.dtype, device=B.device)
    lib = load()
    args = (sten_nmg(n, m, g), _dt(B), values.data_ptr(), idx.data_ptr(), M, K, B.data_ptr(), _ld(B), N,
            out.data_ptr(), _ld(out), _dt(out))
    if plan is None:
        _check(lib.sten_spmm_grouped_nm(*args, _stream(stream)), "sten_spmm_grouped_nm")
    else:
        _check(lib.sten_spmm_grouped_nm_ex(*args, ctypes.byref(plan), _stream(stream)), "sten_spmm_grouped_nm_ex")
    return out


def spmm_autotune(values: torch.Tensor, idx: torch.Tensor, B: torch.Tensor, n: int, m: int, g: int,
                  out: torch.Tensor, reps: int = 5, stream=None) -> sten_spmm_plan:
    """Fastest compiled plan for this shape, measured on the device (out is scratch)."""
    _check_operands(values, idx, B)
    M = values.shape[0]
    K, N = B.shape
    plan = sten_spmm_plan()
    _check(load().sten_spmm_autotune(sten_nmg(n, m, g), _dt(B), values.data_ptr(), idx.data_ptr(), M, K,
                                     B.data_ptr(), _ld(B), N, out.data_ptr(), _ld(out), _dt(out), int(reps),
                                     _stream(stream), ctypes.byref(plan)), "sten_spmm_autotune")
    return plan


def spmm_grouped_nm_allgather(values: torch.Tensor, idx: torch.Tensor, B: torch.Tensor, n: int, m: int, g: int,
                              outs, col0: int, plan: sten_spmm_plan | None = None, stream=None):
    """C_loc = densify(values, idx) @ B written by the SpMM epilogue into columns [col0, col0 + N) of
    EVERY buffer in `outs` (the gathered [M][ldc] outputs of all ranks: peer-mapped views, or
    local tensors) -- sten_spmm_grouped_nm_allgather."""
    _check_operands(values, idx, B)
    M = values.shape[0]
    K, N = B.shape
    ld = _ld(outs[0])
    if any(_ld(o) != ld or o.dtype != outs[0].dtype or o.shape[0] != M for o in outs):
        raise ValueError("every gathered output must share shape, ld and dtype")
    ptrs = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
    _check(load().sten_spmm_grouped_nm_allgather(
        sten_nmg(n, m, g), _dt(values), values.data_ptr(), idx.data_ptr(), M, K, B.data_ptr(), _ld(B), N,
        ptrs, len(outs), col0, ld, _dt(outs[0]), ctypes.byref(plan) if plan is not None else None,
        _stream(stream)), "sten_spmm_grouped_nm_allgather")
    return outs


def spmm_grouped_nm_batched(problems, tile: int = 1, stream=None):
    """ONE launch for several independent fp32 problems: problems = [(values, idx, B, n, m, g, C), ...];
    each C [M][N] receives densify(values, idx) @ B (sten_spmm_grouped_nm_batched)."""
    arr = (sten_spmm_problem * len(problems))()
    for k, (values, idx, B, n, m, g, C) in enumerate(problems):
        _check_operands(values, idx, B)
        arr[k].f = sten_nmg(n, m, g)
        arr[k].values, arr[k].idx = values.data_ptr(), idx.data_ptr()
        arr[k].M, arr[k].K = values.shape[0], B.shape[0]
        arr[k].B, arr[k].ldb, arr[k].N = B.data_ptr(), _ld(B), B.shape[1]
        arr[k].C, arr[k].ldc = C.data_ptr(), _ld(C)
        if values.dtype != torch.float32 or B.dtype != torch.float32 or C.dtype != torch.float32:
            raise TypeError("the grouped launch is fp32")
    _check(load().sten_spmm_grouped_nm_batched(len(problems), arr, tile, _stream(stream)),
           "sten_spmm_grouped_nm_batched")
    return [p[6] for p in problems]


def _problem_array(problems):
    arr = (sten_spmm_problem * len(problems))()
    for k, (values, idx, B, n, m, g, C) in enumerate(problems):
        _check_operands(values, idx, B)
        arr[k].f = sten_nmg(n, m, g)
        arr[k].values, arr[k].idx = values.data_ptr(), idx.data_ptr()
        arr[k].M, arr[k].K = values.shape[0], B.shape[0]
        arr[k].B, arr[k].ldb, arr[k].N = B.data_ptr(), _ld(B), B.shape[1]
        arr[k].C, arr[k].ldc = C.data_ptr(), _ld(C)
        if values.dtype != torch.float32 or B.dtype != torch.float32 or C.dtype != torch.float32:
            raise TypeError("the grouped launch is fp32")
    return arr


def batched_workspace_size(problems, splits=None, tile: int = 1) -> int:
    arr = _problem_array(problems)
    sp = (ctypes.c_int32 * len(problems))(*splits) if splits is not None else None
    nb = _i64()
    _check(load().sten_spmm_batched_workspace_size(len(problems), arr, sp, tile, ctypes.byref(nb)),
           "sten_spmm_batched_workspace_size")
    return nb.value


def spmm_grouped_nm_batched_ex(problems, workspace: torch.Tensor | None, splits=None, tile: int = 1, stream=None):
    """ONE launch for several independent fp32 problems WITH per-problem split-K (splits None = automatic),
    partials reduced through `workspace` (zero-filled once at allocation; sten_spmm_grouped_nm_batched_ex)."""
    arr = _problem_array(problems)
    sp = (ctypes.c_int32 * len(problems))(*splits) if splits is not None else None
    ws_ptr = workspace.data_ptr() if workspace is not None else None
    ws_bytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    _check(load().sten_spmm_grouped_nm_batched_ex(len(problems), arr, sp, tile, ws_ptr, ws_bytes, _stream(stream)),
           "sten_spmm_grouped_nm_batched_ex")
    return [p[6] for p in problems]


ACT_NONE, ACT_GELU, ACT_RELU = 0, 1, 2


def spmm_grouped_nm_bias_act(values: torch.Tensor, idx: torch.Tensor, B: torch.Tensor, n: int, m: int, g: int,
                             bias: torch.Tensor | None = None, act: int = ACT_GELU, out: torch.Tensor | None = None,
                             out_dtype=None, plan: sten_spmm_plan | None = None, stream=None) -> torch.Tensor:
    """C = act(densify(values, idx) @ B + bias[:, None]) with the bias/activation in the SpMM epilogue."""
    _check_operands(values, idx, B)
    M = values.shape[0]
    K, N = B.shape
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype or values.dtype, device=B.device)
    if bias is not None and (bias.dtype != torch.float32 or bias.numel() != M or not bias.is_contiguous()):
        raise ValueError("bias must be a contiguous float32 vector of length M")
    _check(load().sten_spmm_grouped_nm_bias_act(
        sten_nmg(n, m, g), _dt(values), values.data_ptr(), idx.data_ptr(), M, K, B.data_ptr(), _ld(B), N,
        out.data_ptr(), _ld(out), _dt(out), bias.data_ptr() if bias is not None else None, act,
        ctypes.byref(plan) if plan is not None else None, _stream(stream)), "sten_spmm_grouped_nm_bias_act")
    return out


def spmm_grouped_nm_epilogue(values: torch.Tensor, idx: torch.Tensor, B: torch.Tensor, n: int, m: int, g: int,
                             bias: torch.Tensor | None = None, act: int = ACT_NONE,
                             residual: torch.Tensor | None = None, out: torch.Tensor | None = None, out_dtype=None,
                             plan: sten_spmm_plan | None = None, stream=None) -> torch.Tensor:
    """C = act(densify(values, idx) @ B + bias[:, None]) + residual, all in the SpMM epilogue."""
    _check_operands(values, idx, B)
    M = values.shape[0]
    K, N = B.shape
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype or values.dtype, device=B.device)
    if bias is not None and (bias.dtype != torch.float32 or bias.numel() != M or not bias.is_contiguous()):
        raise ValueError("bias must be a contiguous float32 vector of length M")
    if residual is not None and (residual.dtype != out.dtype or tuple(residual.shape) != (M, N)):
        raise ValueError("residual must be [M][N] in the output dtype")
    _check(load().sten_spmm_grouped_nm_epilogue(
        sten_nmg(n, m, g), _dt(values), values.data_ptr(), idx.data_ptr(), M, K, B.data_ptr(), _ld(B), N,
        out.data_ptr(), _ld(out), _dt(out), bias.data_ptr() if bias is not None else None, act,
        residual.data_ptr() if residual is not None else None, _ld(residual) if residual is not None else 0,
        ctypes.byref(plan) if plan is not None else None, _stream(stream)), "sten_spmm_grouped_nm_epilogue")
    return out


def sparse_linear_host(W_host: torch.Tensor, B_host: torch.Tensor, n: int, m: int, g: int,
                       C_host: torch.Tensor, workspace: torch.Tensor, stream=None) -> torch.Tensor:
    """End-to-end: host W, host B -> host C through sten_sparse_linear_host (blocking)."""
    M, K = W_host.shape
    N = B_host.shape[1]
    _check(load().sten_sparse_linear_host(sten_nmg(n, m, g), _dt(W_host), W_host.data_ptr(), M, K, _ld(W_host),
                                          B_host.data_ptr(), _ld(B_host), N, C_host.data_ptr(), _ld(C_host),
                                          _dt(C_host), workspace.data_ptr(), workspace.numel(), _stream(stream)),
           "sten_sparse_linear_host")
    return C_host


def sparse_linear_host_async(W_host: torch.Tensor, B_host: torch.Tensor, n: int, m: int, g: int,
                             C_host: torch.Tensor, workspace: torch.Tensor, stream=None) -> torch.Tensor:
    """sten_sparse_linear_host_async: enqueue H2D, sparsify, SpMM, D2H on `stream`; no wait
    (pinned host buffers; C_host is valid once the stream has drained)."""
    M, K = W_host.shape
    N = B_host.shape[1]
    _check(load().sten_sparse_linear_host_async(sten_nmg(n, m, g), _dt(W_host), W_host.data_ptr(), M, K,
                                                _ld(W_host), B_host.data_ptr(), _ld(B_host), N, C_host.data_ptr(),
                                                _ld(C_host), _dt(C_host), workspace.data_ptr(), workspace.numel(),
                                                _stream(stream)), "sten_sparse_linear_host_async")
    return C_host


def sparse_linear_host_pipelined_async(problems, copy_in, compute, copy_out):
    """sten_sparse_linear_host_pipelined_async: problems = [(W_host, B_host, n, m, g, C_host, workspace), ...];
    H2D on copy_in back to back, kernels on compute, D2H on copy_out, handed over by events (no wait)."""
    arr = (sten_host_linear_problem * len(problems))()
    ab = c = None
    for k, (W_host, B_host, n, m, g, C_host, workspace) in enumerate(problems):
        ab = ab if ab is not None else _dt(W_host)
        c = c if c is not None else _dt(C_host)
        if _dt(W_host) != ab or _dt(B_host) != ab or _dt(C_host) != c:
            raise TypeError("one dtype for every W / B, one for every C")
        arr[k].f = sten_nmg(n, m, g)
        arr[k].W_host, arr[k].M, arr[k].K, arr[k].ldw = W_host.data_ptr(), W_host.shape[0], W_host.shape[1], _ld(W_host)
        arr[k].B_host, arr[k].ldb, arr[k].N = B_host.data_ptr(), _ld(B_host), B_host.shape[1]
        arr[k].C_host, arr[k].ldc = C_host.data_ptr(), _ld(C_host)
        arr[k].workspace, arr[k].workspace_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    _check(load().sten_sparse_linear_host_pipelined_async(len(problems), arr, ab, c, _stream(copy_in),
                                                          _stream(compute), _stream(copy_out)),
           "sten_sparse_linear_host_pipelined_async")
    return [p[5] for p in problems]


def sparse_linear_host_workspace_size(n: int, m: int, g: int, M: int, K: int, N: int,
                                      ab_dtype=torch.float32, c_dtype=torch.float32) -> int:
    return int(load().sten_sparse_linear_host_workspace_size(
        sten_nmg(n, m, g), F32 if ab_dtype == torch.float32 else BF16, M, K, N,
        F32 if c_dtype == torch.float32 else BF16))


def launch_count(plan: sten_spmm_plan) -> int:
    return int(load().sten_spmm_launch_count(ctypes.byref(plan)))


def algo_name(algo: int) -> str:
    return load().sten_algo_name(algo).decode()


def status_string(s: int) -> str:
    return load().sten_status_string(s).decode()


# ---------------------------------------------------------------------------------------------
# Chunked n:m:g -- the paper's own format (include/sten.h "Chunked n:m:g")
# ---------------------------------------------------------------------------------------------
def nmg_chunk(n: int, m: int, g: int) -> int:
    """L = C(m, n) g columns per chunk."""
    return math.comb(m, n) * g


NMG_GREEDY, NMG_EXCHANGE, NMG_GREEDY_EXCHANGE = 0, 1, 2


def nmg_sparsify(W: torch.Tensor, n: int, m: int, g: int, values: torch.Tensor | None = None,
                 idx: torch.Tensor | None = None, stream=None, method: int = NMG_GREEDY):
    """dense W [M][K] -> (values [M/m][K/L][L][n], idx [M/m][K/L][L] int16 bit patterns of uint16);
    method: 0 greedy, 1 the paper's GPU exchange conversion, 2 greedy + exchange (sten_nmg_sparsify_ex)."""
    _cuda(W, "W")
    M, K = W.shape
    L = nmg_chunk(n, m, g)
    if values is None:
        values = torch.empty((M // m, K // L, L, n), dtype=W.dtype, device=W.device)
    if idx is None:
        idx = torch.empty((M // m, K // L, L), dtype=torch.int16, device=W.device)
    _check(load().sten_nmg_sparsify_ex(sten_nmg(n, m, g), _dt(W), W.data_ptr(), M, K, _ld(W),
                                       values.data_ptr(), idx.data_ptr(), int(method), _stream(stream)),
           "sten_nmg_sparsify_ex")
    return values, idx


def nmg_densify(values: torch.Tensor, idx: torch.Tensor, n: int, m: int, g: int, K: int,
                out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    M = values.shape[0] * m
    if out is None:
        out = torch.empty((M, K), dtype=values.dtype, device=values.device)
    _check(load().sten_nmg_densify(sten_nmg(n, m, g), _dt(values), values.data_ptr(), idx.data_ptr(), M, K,
                                   out.data_ptr(), _ld(out), _stream(stream)), "sten_nmg_densify")
    return out


def nmg_spmm(values: torch.Tensor, idx: torch.Tensor, B: torch.Tensor, n: int, m: int, g: int,
             out: torch.Tensor | None = None, out_dtype=None, stream=None) -> torch.Tensor:
    """C [M][N] = densify(values, idx) @ B [K][N] (chunked n:m:g)."""
    _cuda(B, "B")
    M = values.shape[0] * m
    K, N = B.shape
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype or values.dtype, device=B.device)
    _check(load().sten_nmg_spmm(sten_nmg(n, m, g), _dt(values), values.data_ptr(), idx.data_ptr(), M, K,
                                B.data_ptr(), _ld(B), N, out.data_ptr(), _ld(out), _dt(out), _stream(stream)),
           "sten_nmg_spmm")
    return out


# ---- K6: 2:4 structured-sparse tensor-core path (NEXT-4) --------------------------------------

def sp24_compatible(n: int, m: int) -> bool:
    """Grouped n:m formats whose every pattern is 2:4 on aligned 4-windows of K."""
    return n == 1 or (n == 2 and m % 4 == 0)


def sp24_pack(values: torch.Tensor, idx: torch.Tensor, n: int, m: int, g: int, K: int, stream=None,
              v24: torch.Tensor | None = None, meta: torch.Tensor | None = None):
    """(values, idx) -> (v24 [M128][K128/2] bf16, meta uint32) for sten_spmm_sp24 (sten_sp24_pack);
    v24 / meta may be preallocated (shapes of an earlier call)."""
    _cuda(values, "values")
    if values.dtype != torch.bfloat16 or idx.dtype != torch.uint8:
        raise TypeError("sp24 packs bf16 values with uint8 idx")
    M = values.shape[0]
    vb, mb = _i64(), _i64()
    lib = load()
    _check(lib.sten_sp24_packed_size(sten_nmg(n, m, g), M, K, ctypes.byref(vb), ctypes.byref(mb)),
           "sten_sp24_packed_size")
    M128 = -(-M // 128) * 128
    if v24 is None:
        v24 = torch.empty((M128, vb.value // 2 // max(M128, 1)), dtype=torch.bfloat16, device=values.device)
    if meta is None:
        meta = torch.empty((mb.value // 4,), dtype=torch.int32, device=values.device)
    if v24.numel() * 2 < vb.value or meta.numel() * 4 < mb.value:
        raise ValueError("preallocated v24 / meta too small")
    _check(lib.sten_sp24_pack(sten_nmg(n, m, g), BF16, values.data_ptr(), idx.data_ptr(), M, K, v24.data_ptr(),
                              meta.data_ptr(), _stream(stream)), "sten_sp24_pack")
    return v24, meta


def spmm_sp24(v24: torch.Tensor, meta: torch.Tensor, M: int, K: int, B: torch.Tensor,
              out: torch.Tensor | None = None, out_dtype=None, tile: int = 0, stream=None) -> torch.Tensor:
    """C [M][N] = densify(values, idx) @ B on the 2:4 sparse tensor cores (sten_spmm_sp24)."""
    _cuda(B, "B")
    if B.dtype != torch.bfloat16:
        raise TypeError("sten_spmm_sp24 takes bf16 B")
    N = B.shape[1]
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype or torch.bfloat16, device=B.device)
    _check(load().sten_spmm_sp24(v24.data_ptr(), meta.data_ptr(), M, K, B.data_ptr(), _ld(B), N, out.data_ptr(),
                                 _ld(out), _dt(out), int(tile), _stream(stream)), "sten_spmm_sp24")
    return out


def spmm_sp24_epilogue(v24: torch.Tensor, meta: torch.Tensor, M: int, K: int, B: torch.Tensor,
                       bias: torch.Tensor | None = None, act: int = 0, residual: torch.Tensor | None = None,
                       out: torch.Tensor | None = None, out_dtype=None, tile: int = 0, stream=None) -> torch.Tensor:
    """C = act(densify @ B + bias[:, None]) + residual on the 2:4 sparse tensor cores (sten_spmm_sp24_epilogue)."""
    _cuda(B, "B")
    if B.dtype != torch.bfloat16:
        raise TypeError("sten_spmm_sp24 takes bf16 B")
    N = B.shape[1]
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype or torch.bfloat16, device=B.device)
    if bias is not None and (bias.dtype != torch.float32 or bias.numel() != M or not bias.is_contiguous()):
        raise ValueError("bias must be a contiguous float32 vector of length M")
    if residual is not None and (residual.dtype != out.dtype or tuple(residual.shape) != (M, N)):
        raise ValueError("residual must be [M][N] in the output dtype")
    _check(load().sten_spmm_sp24_epilogue(
        v24.data_ptr(), meta.data_ptr(), M, K, B.data_ptr(), _ld(B), N, out.data_ptr(), _ld(out), _dt(out),
        bias.data_ptr() if bias is not None else None, int(act),
        residual.data_ptr() if residual is not None else None, _ld(residual) if residual is not None else 0,
        int(tile), _stream(stream)), "sten_spmm_sp24_epilogue")
    return out
