"""NEXT-3: a BERT-base encoder whose linear layers run on the grouped n:m kernels (PAPER.md:720-730,
section 6.2 "Sparse inference": the paper's BERT-base inference with n:m:g linears).

Activations are kept FEATURE-MAJOR, x^T [hidden][tokens], the layout the SpMM consumes (B = x^T,
C = y^T), so the four linears of a layer chain without transposes:

    qkv^T = Wqkv . x^T + bqkv                                   (SpMM, bias in the epilogue)
    a     = softmax(q k^T / sqrt(d)) v                          (torch SDPA, per head)
    h^T   = LN(Wo . a^T + bo + x^T)                             (SpMM, bias + residual in the epilogue)
    f^T   = GELU(W1 . h^T + b1)                                 (SpMM, bias + GELU in the epilogue)
    y^T   = LN(W2 . f^T + b2 + h^T)                             (SpMM, bias + residual in the epilogue)

Attention (SDPA) and LayerNorm run as torch ops (layout copies around SDPA are device-memory
plumbing); every linear is ONE launch of the library's SpMM with its epilogue fused: the SIMT kernel
(fp32), or for bf16 with a 2:4-compatible format the 2:4 structured-sparse tensor-core kernel (K6,
weights packed once at load).  The dense
reference (`DenseBertLayer`) is the same layer with cuBLAS GEMMs on densify(W) -- the GPU analogue
of the paper's "vs dense PyTorch" comparison.
"""
from __future__ import annotations

import math

import torch
import torch.nn.functional as F

from . import sten

HIDDEN, HEADS, FFN = 768, 12, 3072


def layer_norm_fm(h: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, eps: float = 1e-12) -> torch.Tensor:
    """LayerNorm over the feature dimension (dim 0) of a feature-major activation [H][N]."""
    mean = h.mean(0, keepdim=True)
    var = (h - mean).pow(2).mean(0, keepdim=True)
    return (h - mean) * torch.rsqrt(var + eps) * gamma[:, None] + beta[:, None]


def attention_fm(qkv: torch.Tensor, batch: int, seq: int) -> torch.Tensor:
    """qkv^T [3 H][N] feature-major (N = batch * seq, tokens batch-major) -> a^T [H][N]."""
    d = HIDDEN // HEADS
    t = qkv.view(3, HEADS, d, batch, seq).permute(0, 3, 1, 4, 2)          # [3][B][heads][S][d]
    q, k, v = (t[i].contiguous() for i in range(3))
    a = F.scaled_dot_product_attention(q, k, v)                           # [B][heads][S][d]
    return a.permute(1, 3, 0, 2).reshape(HIDDEN, batch * seq).contiguous()


def random_layer_weights(seed: int, device) -> dict:
    """BERT-base layer parameters (random init at the BERT scale: N(0, 0.02^2), zero-ish biases, LN = 1/0)."""
    gen = torch.Generator(device="cpu").manual_seed(seed)

    def w(o, i):
        return (torch.randn(o, i, generator=gen) * 0.02).to(device)

    def b(o):
        return (torch.randn(o, generator=gen) * 0.02).to(device)

    return {"qkv": w(3 * HIDDEN, HIDDEN), "bqkv": b(3 * HIDDEN), "o": w(HIDDEN, HIDDEN), "bo": b(HIDDEN),
            "ln1_g": torch.ones(HIDDEN, device=device), "ln1_b": torch.zeros(HIDDEN, device=device),
            "w1": w(FFN, HIDDEN), "b1": b(FFN), "w2": w(HIDDEN, FFN), "b2": b(HIDDEN),
            "ln2_g": torch.ones(HIDDEN, device=device), "ln2_b": torch.zeros(HIDDEN, device=device)}


class SparseBertLayer:
    """One encoder layer with its four linears in grouped n:m form (sparsified once, at load)."""

    def __init__(self, wts: dict, n: int, m: int, g: int, dtype=torch.float32, backend: str | None = None):
        self.fmt = (n, m, g)
        self.dtype = dtype
        # bf16 with a 2:4-compatible format -> the 2:4 structured-sparse tensor cores (K6, fused epilogue);
        # otherwise the SIMT SpMM with its fused epilogue
        self.backend = backend or ("sp24" if dtype == torch.bfloat16 and sten.sp24_compatible(n, m) else "simt")
        self.lin = {}
        self.packed = {}
        for name in ("qkv", "o", "w1", "w2"):
            W = wts[name].to(dtype).contiguous()
            self.lin[name] = sten.sparsify_grouped_nm(W, n, m, g)
            if self.backend == "sp24":
                self.packed[name] = sten.sp24_pack(*self.lin[name], n, m, g, W.shape[1])
        self.bias = {k: wts[k].float().contiguous() for k in ("bqkv", "bo", "b1", "b2")}
        self.ln = {k: wts[k].to(dtype) for k in ("ln1_g", "ln1_b", "ln2_g", "ln2_b")}

    def dense_weights(self) -> dict:
        """densify(values, idx) of every linear (the masked weights, for the dense reference)."""
        n, m, g = self.fmt
        out = {}
        for name, (v, i) in self.lin.items():
            out[name] = sten.densify(v, i, n, m, g, i.shape[1] * m)
        return out

    def _linear(self, name: str, B: torch.Tensor, bias, act: int = 0, residual=None) -> torch.Tensor:
        n, m, g = self.fmt
        if self.backend == "sp24":
            v24, meta = self.packed[name]
            return sten.spmm_sp24_epilogue(v24, meta, self.lin[name][0].shape[0], B.shape[0], B, bias=bias, act=act,
                                           residual=residual, out_dtype=self.dtype)
        return sten.spmm_grouped_nm_epilogue(*self.lin[name], B, n, m, g, bias=bias, act=act, residual=residual)

    def __call__(self, xT: torch.Tensor, batch: int, seq: int) -> torch.Tensor:
        qkv = self._linear("qkv", xT, self.bias["bqkv"])
        aT = attention_fm(qkv, batch, seq)
        h = self._linear("o", aT, self.bias["bo"], residual=xT)
        h = layer_norm_fm(h, self.ln["ln1_g"], self.ln["ln1_b"]).contiguous()
        f = self._linear("w1", h, self.bias["b1"], act=sten.ACT_GELU)
        y = self._linear("w2", f, self.bias["b2"], residual=h)
        return layer_norm_fm(y, self.ln["ln2_g"], self.ln["ln2_b"]).contiguous()


class DenseBertLayer:
    """The same layer with dense cuBLAS GEMMs on the given weights (e.g. densify(W) of a sparse layer)."""

    def __init__(self, dense: dict, sparse: SparseBertLayer):
        self.w = {k: v.contiguous() for k, v in dense.items()}
        self.bias = {k: v.to(sparse.dtype) for k, v in sparse.bias.items()}
        self.ln = sparse.ln

    def __call__(self, xT: torch.Tensor, batch: int, seq: int) -> torch.Tensor:
        qkv = torch.addmm(self.bias["bqkv"][:, None], self.w["qkv"], xT)
        aT = attention_fm(qkv, batch, seq)
        h = torch.addmm(self.bias["bo"][:, None], self.w["o"], aT) + xT
        h = layer_norm_fm(h, self.ln["ln1_g"], self.ln["ln1_b"]).contiguous()
        f = F.gelu(torch.addmm(self.bias["b1"][:, None], self.w["w1"], h))
        y = torch.addmm(self.bias["b2"][:, None], self.w["w2"], f) + h
        return layer_norm_fm(y, self.ln["ln2_g"], self.ln["ln2_b"]).contiguous()


class Encoder:
    """A stack of layers; `capture` records the whole forward in ONE CUDA graph (static input/output)."""

    def __init__(self, layers):
        self.layers = layers
        self.graph = None

    def __call__(self, xT: torch.Tensor, batch: int, seq: int) -> torch.Tensor:
        for lyr in self.layers:
            xT = lyr(xT, batch, seq)
        return xT

    def capture(self, xT_static: torch.Tensor, batch: int, seq: int):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                self(xT_static, batch, seq)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.out_static = self(xT_static, batch, seq)
        return self.out_static

    def replay(self):
        self.graph.replay()
        return self.out_static


def attention_flops(batch: int, seq: int) -> float:
    return 4.0 * batch * seq * seq * HIDDEN


def linear_flops(tokens: int) -> float:
    """dense-equivalent flops of the four linears of one layer."""
    return 2.0 * tokens * (3 * HIDDEN * HIDDEN + HIDDEN * HIDDEN + 2 * HIDDEN * FFN)


__all__ = ["SparseBertLayer", "DenseBertLayer", "Encoder", "random_layer_weights", "layer_norm_fm", "attention_fm",
           "linear_flops", "attention_flops", "math"]
