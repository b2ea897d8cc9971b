"""GPU parity of NEXT-2 (masked linear training path with a fixed mask; the
fixed-mask fast path) against the CPU oracle.

  * SDDMM (weight gradient in the values layout): rel err |dV - dV_ref| / Bound <= 1e-5 (fp32),
    2e-2 (bf16); integer inputs bit-exact; deterministic (two runs equal bit for bit);
  * mask check + re-pack: values bit-exact, outside count exact;
  * GroupedNMLinear forward / backward vs the oracle (forward SpMM, SDDMM, dx = dy densify(W)).
"""
import numpy as np
import pytest
import torch

import oracle
import synthetic
from paper_2304_07613_b200 import sten
from paper_2304_07613_b200.masked_linear import GroupedNMLinear
from test_gpu_parity import dev, host

pytestmark = pytest.mark.gpu

FMT = [(2, 4, 4), (1, 4, 1), (1, 10, 2), (3, 6, 3), (2, 8, 8), (1, 2, 2), (2, 4, 16)]


def rel(x, ref, bound):
    x = x.detach().float().cpu().numpy().astype(np.float64)
    return float(np.max(np.abs(x - ref) / np.maximum(bound, 1e-30))) if x.size else 0.0


@pytest.mark.parametrize("n,m,g", FMT)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("N", [1, 37, 700])
def test_sddmm_vs_oracle(n, m, g, dtype, N):
    M, K = 24 * g if g < 8 else 5 * g, 13 * m
    W = synthetic.weights(M, K, seed=n + m + g, dtype=dtype)
    B = synthetic.activations(K, N, seed=N + 1, dtype=dtype)
    G = synthetic.activations(M, N, seed=N + 2, dtype=dtype)
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    dV_ref, bound = oracle.sddmm(G, B, i_ref, n, m, g, nthreads=oracle.max_threads())
    v, i = sten.sparsify_grouped_nm(dev(W, dtype), n, m, g)
    dV = sten.sddmm_grouped_nm(dev(G, dtype), dev(B, dtype), i, n, m, g, out_dtype=torch.float32)
    dV2 = sten.sddmm_grouped_nm(dev(G, dtype), dev(B, dtype), i, n, m, g, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(dV, dV2)                                  # deterministic
    assert rel(dV, dV_ref, bound) <= (1e-5 if dtype == "f32" else 2e-2)


@pytest.mark.parametrize("n,m,g", FMT[:4])
def test_sddmm_integer_exact(n, m, g):
    M, K, N = 8 * g, 9 * m, 257
    W = synthetic.integer_matrix(M, K, seed=1)
    B = synthetic.integer_matrix(K, N, seed=2, lo=-3, hi=3)
    G = synthetic.integer_matrix(M, N, seed=3, lo=-3, hi=3)
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    dV_ref, _ = oracle.sddmm(G, B, i_ref, n, m, g)
    v, i = sten.sparsify_grouped_nm(dev(W, "f32"), n, m, g)
    dV = sten.sddmm_grouped_nm(dev(G, "f32"), dev(B, "f32"), i, n, m, g)
    torch.cuda.synchronize()
    assert np.array_equal(dV.cpu().numpy().astype(np.float64), dV_ref)


@pytest.mark.parametrize("n,m,g", FMT)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_mask_check_repack(n, m, g, dtype):
    M, K = 8 * g, 10 * m
    W = synthetic.weights(M, K, seed=5, dtype=dtype)
    v, i = sten.sparsify_grouped_nm(dev(W, dtype), n, m, g)
    D = sten.densify(v, i, n, m, g, K)
    vals, out = sten.mask_check_repack(D, i, n, m, g)
    torch.cuda.synchronize()
    assert int(out.item()) == 0 and torch.equal(vals, v)
    W2 = synthetic.weights(M, K, seed=6, dtype=dtype)
    W2h = W2.copy()
    W2h[np.random.default_rng(0).random((M, K)) < 0.3] = 0
    ref_vals, ref_out = oracle.mask_check(W2h, host(i), n, m, g)
    vals, out = sten.mask_check_repack(dev(W2h, dtype), i, n, m, g)
    torch.cuda.synchronize()
    assert int(out.item()) == ref_out
    assert np.array_equal(host(vals).view(np.uint8), ref_vals.view(np.uint8))


@pytest.mark.parametrize("n,m,g", [(2, 4, 4), (1, 10, 2), (2, 8, 8)])
@pytest.mark.parametrize("with_bias", [True, False])
def test_grouped_nm_linear_forward_backward(n, m, g, with_bias):
    """y = x W^T + b and its gradients through autograd, against the oracle in fp64."""
    Ntok, K, M = 300, 12 * m, 16 * g
    W = synthetic.weights(M, K, seed=11)
    x = synthetic.activations(Ntok, K, seed=12)              # [N][K] token-major
    gy = synthetic.activations(Ntok, M, seed=13)
    b = (np.random.default_rng(4).standard_normal(M) * 0.1).astype(np.float32)
    lin = GroupedNMLinear.from_dense(torch.from_numpy(W).cuda(), n, m, g,
                                     bias=torch.from_numpy(b).cuda() if with_bias else None)
    xt = torch.from_numpy(x).cuda().requires_grad_(True)
    y = lin(xt)
    y.backward(torch.from_numpy(gy).cuda())
    torch.cuda.synchronize()
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    B = np.ascontiguousarray(x.T)
    C_ref, Cb = oracle.spmm(v_ref, i_ref, B, n, m, g)
    y_ref = C_ref.T + (b[None, :].astype(np.float64) if with_bias else 0.0)
    assert rel(y, y_ref, Cb.T + (np.abs(b)[None, :] if with_bias else 0)) <= 1e-5
    dV_ref, dVb = oracle.sddmm(np.ascontiguousarray(gy.T), B, i_ref, n, m, g)
    assert rel(lin.values.grad, dV_ref, dVb) <= 1e-5
    Wm = oracle.densify(v_ref, i_ref, n, m, g, K).astype(np.float64)
    dx_ref = gy.astype(np.float64) @ Wm
    dx_bound = np.abs(gy.astype(np.float64)) @ np.abs(Wm)
    assert rel(xt.grad, dx_ref, dx_bound) <= 1e-5
    if with_bias:
        assert rel(lin.bias.grad, gy.astype(np.float64).sum(0), np.abs(gy.astype(np.float64)).sum(0)) <= 1e-5
    # an optimizer step on the values keeps the mask: load_dense of the new dense weight reports 0 outside
    with torch.no_grad():
        lin.values -= 0.1 * lin.values.grad
    assert lin.load_dense(lin.dense_weight()) == 0
