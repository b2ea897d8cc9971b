"""NEXT-2: the grouped n:m linear layer for sparse fine-tuning / training with a FIXED mask
(STen's FixedMaskTensor path) on the C-ABI kernels.

    y = x W_masked^T + b        W_masked = densify(values, idx)      (x [N][K], y [N][M])

* forward: the grouped n:m SpMM (sten_spmm_grouped_nm / _bias_act), C = y^T = densify(values, idx) x^T;
* backward:
    dvalues = (dy^T x) sampled at the kept positions -- the weight gradient in the SAME format
              (sten_sddmm_grouped_nm; the "(KeepAll, FixedMaskTensor)" gradient of PAPER.md:606-617),
    dx      = dy W_masked  -- the paper's masked-dense training path ("Linear operators will use
              masked dense tensors during training"): densify (our kernel) + a plain
              library GEMM,
    dbias   = sum_tokens dy;
* optimizer steps update `values` in place: the mask never changes, so no re-sparsification is
  needed (the fixed-mask fast path); a dense weight arriving from elsewhere (e.g. a
  gradient all-reduce in dense form) is re-packed with `load_dense`, which also reports whether its
  nonzeros still match the mask (sten_mask_check_repack).

Transposes between the torch token-major layout and the kernels' [K][N] operand are layout copies
(device-memory plumbing); every arithmetic step runs in the library's kernels or cuBLAS.
"""
from __future__ import annotations

import torch

from . import sten


class GroupedNMLinearFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, values, idx, bias, n, m, g):
        B = x.t().contiguous()                                       # [K][N]
        if bias is not None:
            C = sten.spmm_grouped_nm_bias_act(values, idx, B, n, m, g, bias=bias.float().contiguous(),
                                              act=sten.ACT_NONE)
        else:
            C = sten.spmm_grouped_nm(values, idx, B, n, m, g)
        ctx.save_for_backward(B, values, idx)
        ctx.fmt = (n, m, g)
        ctx.has_bias = bias is not None
        return C.t()

    @staticmethod
    def backward(ctx, gy):
        B, values, idx = ctx.saved_tensors
        n, m, g = ctx.fmt
        G = gy.t().contiguous().to(values.dtype)                     # [M][N]
        dvalues = sten.sddmm_grouped_nm(G, B, idx, n, m, g, out_dtype=values.dtype)
        dx = None
        if ctx.needs_input_grad[0]:
            W = sten.densify(values, idx, n, m, g, B.shape[0])
            dx = gy.to(values.dtype) @ W
        dbias = gy.sum(0) if ctx.has_bias else None
        return dx, dvalues, None, dbias, None, None, None


class GroupedNMLinear(torch.nn.Module):
    """Linear layer whose weight is stored in grouped n:m form with a fixed mask."""

    def __init__(self, values: torch.Tensor, idx: torch.Tensor, n: int, m: int, g: int, K: int,
                 bias: torch.Tensor | None = None):
        super().__init__()
        self.n, self.m, self.g, self.in_features = n, m, g, K
        self.values = torch.nn.Parameter(values)
        self.register_buffer("idx", idx)
        self.bias = torch.nn.Parameter(bias) if bias is not None else None

    @classmethod
    def from_dense(cls, weight: torch.Tensor, n: int, m: int, g: int, bias: torch.Tensor | None = None):
        """GroupedNMSparsifier(n, m, g): magnitude sparsification of a dense weight."""
        v, i = sten.sparsify_grouped_nm(weight.detach().contiguous(), n, m, g)
        return cls(v, i, n, m, g, weight.shape[1], None if bias is None else bias.detach().clone())

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return GroupedNMLinearFunction.apply(x, self.values, self.idx, self.bias, self.n, self.m, self.g)

    def dense_weight(self) -> torch.Tensor:
        return sten.densify(self.values.detach(), self.idx, self.n, self.m, self.g, self.in_features)

    @torch.no_grad()
    def load_dense(self, weight: torch.Tensor) -> int:
        """SameFormatSparsifier with the fixed-mask check: re-pack `weight` at the
        existing pattern; returns the number of its nonzeros outside the mask (0 = the locations
        match, the re-pack is exact)."""
        v, outside = sten.mask_check_repack(weight.contiguous(), self.idx, self.n, self.m, self.g,
                                            values=self.values.data)
        return int(outside.item())
