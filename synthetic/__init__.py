"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

This module holds NONE of the method's arithmetic (no scoring, selection,
compaction or product).  It only draws the inputs the paper's workloads
imply:

* W ~ N(0, 0.02^2)  -- BERT initialiser scale, the weights that get sparsified;
* B ~ N(0, 1)       -- post-LayerNorm activation scale, the dense operand;
* integer-valued variants in [-8, 8] for the exactness tests (P7/P8);
* bf16 inputs are made by rounding the fp32 draw to nearest-even bf16
  BEFORE anything else sees them (reading R11), so the oracle and
  the GPU see identical bytes.

Generator: ``numpy.random.Generator(PCG64(seed))``; the default seed of config
index i is ``1234 + i``.
"""
from __future__ import annotations

import dataclasses

import numpy as np

W_STD = 0.02
B_STD = 1.0


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (round-to-nearest-even) and return uint16 bit patterns."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return rounded.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def _finish(x: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "f32":
        return np.ascontiguousarray(x, dtype=np.float32)
    if dtype == "bf16":
        return f32_to_bf16_bits(x)
    raise ValueError("dtype must be 'f32' or 'bf16'")


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def weights(M: int, K: int, seed: int, dtype: str = "f32", k_pad: int = 0) -> np.ndarray:
    """Dense weight W [M][K + k_pad]; the k_pad trailing columns are zero."""
    w = rng(seed).standard_normal((M, K), dtype=np.float32) * np.float32(W_STD)
    if k_pad:
        w = np.concatenate([w, np.zeros((M, k_pad), np.float32)], axis=1)
    return _finish(w, dtype)


def activations(K: int, N: int, seed: int, dtype: str = "f32", k_pad: int = 0) -> np.ndarray:
    """Dense operand B [K + k_pad][N] (= x^T of a linear layer); padded rows are zero."""
    b = rng(seed + 7919).standard_normal((K, N), dtype=np.float32) * np.float32(B_STD)
    if k_pad:
        b = np.concatenate([b, np.zeros((k_pad, N), np.float32)], axis=0)
    return _finish(b, dtype)


def integer_matrix(rows: int, cols: int, seed: int, lo: int = -8, hi: int = 8,
                   dtype: str = "f32") -> np.ndarray:
    """Integer-valued matrix with entries uniform in [lo, hi] (exact in fp32 and bf16)."""
    x = rng(seed).integers(lo, hi + 1, size=(rows, cols)).astype(np.float32)
    return _finish(x, dtype)


def pad_for(K: int, m: int, n: int = 1) -> int:
    """Zero columns of W / rows of B appended so that m | K and 4 | K/m*n (DESIGN.md
    reading R7): the kept count per row is then a multiple of 4, which keeps every
    values row 16-byte aligned for the TMA path.  The effective GFLOP/s metric
    still counts the true (unpadded) K."""
    p = 0
    while (K + p) % m or ((K + p) // m * n) % 4:
        p += 1
    return p


@dataclasses.dataclass(frozen=True)
class Case:
    """One (shape, format) point of a BASELINE.json config."""
    M: int
    K: int
    N: int
    n: int
    m: int
    g: int
    dtype: str = "f32"

    @property
    def k_pad(self) -> int:
        return pad_for(self.K, self.m, self.n)

    @property
    def Kp(self) -> int:          # padded contraction length
        return self.K + self.k_pad

    @property
    def kept(self) -> int:        # K' = kept entries per row
        return self.Kp // self.m * self.n

    def label(self) -> str:
        return "%dx%dx%d %d:%d:g%d %s" % (self.M, self.K, self.N, self.n, self.m, self.g, self.dtype)


# BASELINE.json "configs", index -> list of cases.
BERT_BASE_LINEARS = [(768, 768), (768, 3072), (3072, 768)]     # (M = out, K = in)
BERT_BASE_SPARSITY = [(2, 4), (1, 4), (1, 10)]                  # 50 / 75 / 90 %
BERT_LARGE_LINEARS = [(1024, 4096), (4096, 1024)]


def config_cases(index: int, g: int = 4, dtype: str = "f32") -> list[Case]:
    if index == 0:
        return [Case(64, 64, 32, 2, 4, 4, "f32")]
    if index == 1:
        return [Case(M, K, 8 * 128, n, m, g, dtype)
                for (M, K) in BERT_BASE_LINEARS for (n, m) in BERT_BASE_SPARSITY]
    if index == 2:
        return [Case(M, K, 32 * 512, n, m, g, "bf16")
                for (M, K) in BERT_LARGE_LINEARS for (n, m) in [(1, 4), (2, 8)]]
    if index == 3:
        # one BERT-base encoder layer's linears (QKV fused, O, FFN1, FFN2), 256 x 128 tokens
        return [Case(M, K, 256 * 128, 2, 4, g, dtype)
                for (M, K) in [(2304, 768), (768, 768), (3072, 768), (768, 3072)]]
    if index == 4:
        return [Case(8192, 8192, 65536, 1, 8, g, dtype)]
    raise IndexError(index)
