"""GPU parity of the chunked n:m:g path (the paper's own format; NEXT-1)
through the C ABI against the CPU oracle (-m gpu).

Bars: idx and values bit-exact; densify bit-exact; C rel err (|C - C_ref| / Bound) <= 1e-5
for fp32 inputs, <= 2e-2 for bf16 inputs; integer-valued inputs bit-exact.
"""
import numpy as np
import pytest
import torch

import oracle
import synthetic
from paper_2304_07613_b200 import sten

pytestmark = pytest.mark.gpu

SPMM_SET = [(1, 2, 1), (1, 2, 4), (1, 4, 4), (2, 4, 1), (2, 4, 4), (1, 8, 2), (1, 8, 4),
            (3, 6, 1), (3, 6, 2), (2, 8, 1), (1, 10, 4)]
CONVERT_ONLY = [(2, 5, 2), (1, 3, 3), (2, 6, 1)]


def dev(x: np.ndarray, dtype: str, ld_multiple: int = 8) -> torch.Tensor:
    x = np.ascontiguousarray(x)
    rows, cols = x.shape
    ld = -(-cols // ld_multiple) * ld_multiple if cols else ld_multiple
    if dtype == "bf16":
        t = torch.zeros((rows, ld), dtype=torch.bfloat16)
        t[:, :cols] = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16)
    else:
        t = torch.zeros((rows, ld), dtype=torch.float32)
        t[:, :cols] = torch.from_numpy(x)
    return t.cuda()[:, :cols]


def host(t: torch.Tensor) -> np.ndarray:
    t = t.cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    if t.dtype == torch.int16:
        return t.numpy().view(np.uint16)
    return t.numpy()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n,m,g", SPMM_SET + CONVERT_ONLY)
def test_nmg_sparsify_densify_bit_exact(dtype, n, m, g):
    L = oracle.nmg_chunk(n, m, g)
    M, K = 5 * m, 3 * L
    W = synthetic.weights(M, K, seed=n * 100 + m * 10 + g, dtype=dtype)
    v_ref, i_ref = oracle.nmg_sparsify(W, n, m, g)
    v, i = sten.nmg_sparsify(dev(W, dtype, ld_multiple=1 if dtype == "f32" else 8), n, m, g)
    torch.cuda.synchronize()
    assert np.array_equal(host(i), i_ref)
    assert np.array_equal(host(v).view(np.uint8), v_ref.view(np.uint8))
    D = sten.nmg_densify(v, i, n, m, g, K)
    assert np.array_equal(host(D).view(np.uint8), oracle.nmg_densify(v_ref, i_ref, n, m, g, K).view(np.uint8))


@pytest.mark.parametrize("n,m,g", SPMM_SET + CONVERT_ONLY)
def test_nmg_sparsify_integer_ties(n, m, g):
    """Many exact ties in the magnitudes: the (column, pattern) tie-break must match."""
    L = oracle.nmg_chunk(n, m, g)
    W = synthetic.integer_matrix(4 * m, 4 * L, seed=n + m + g, lo=-2, hi=2)
    v_ref, i_ref = oracle.nmg_sparsify(W, n, m, g)
    v, i = sten.nmg_sparsify(dev(W, "f32"), n, m, g)
    torch.cuda.synchronize()
    assert np.array_equal(host(i), i_ref) and np.array_equal(host(v), v_ref)


def _spmm(W, B, n, m, g, dtype, out_dtype=None):
    v_ref, i_ref = oracle.nmg_sparsify(W, n, m, g)
    C_ref, Bound = oracle.nmg_spmm(v_ref, i_ref, B, n, m, g, nthreads=oracle.max_threads())
    v, i = sten.nmg_sparsify(dev(W, dtype), n, m, g)
    C = sten.nmg_spmm(v, i, dev(B, dtype), n, m, g, out_dtype=out_dtype)
    torch.cuda.synchronize()
    return C, C_ref, Bound


def rel_err(C, C_ref, Bound):
    c = C.float().cpu().numpy().astype(np.float64)
    return float(np.max(np.abs(c - C_ref) / np.maximum(Bound, 1e-30)))


@pytest.mark.parametrize("n,m,g", SPMM_SET)
@pytest.mark.parametrize("N", [1, 128, 301])
def test_nmg_spmm_f32(n, m, g, N):
    L = oracle.nmg_chunk(n, m, g)
    M, K = 19 * m, max(6, 200 // L) * L            # ragged row blocks vs the CTA, several K stages
    W = synthetic.weights(M, K, seed=3 * n + m + g)
    B = synthetic.activations(K, N, seed=5 * n + m + g)
    C, C_ref, Bound = _spmm(W, B, n, m, g, "f32")
    assert rel_err(C, C_ref, Bound) <= 1e-5


@pytest.mark.parametrize("n,m,g", SPMM_SET)
def test_nmg_spmm_bf16(n, m, g):
    L = oracle.nmg_chunk(n, m, g)
    M, K, N = 8 * m, 8 * L, 200
    W = synthetic.weights(M, K, seed=7 * n + m + g, dtype="bf16")
    B = synthetic.activations(K, N, seed=9 * n + m + g, dtype="bf16")
    C, C_ref, Bound = _spmm(W, B, n, m, g, "bf16", out_dtype=torch.float32)
    assert rel_err(C, C_ref, Bound) <= 2e-2
    Cb, _, _ = _spmm(W, B, n, m, g, "bf16")                 # bf16 output (RNE of the fp32 sum)
    assert rel_err(Cb, C_ref, Bound) <= 2e-2


@pytest.mark.parametrize("n,m,g", SPMM_SET)
def test_nmg_spmm_integer_exact(n, m, g):
    L = oracle.nmg_chunk(n, m, g)
    M, K, N = 16 * m, 10 * L, 133
    W = synthetic.integer_matrix(M, K, seed=n + 2 * m + 3 * g, lo=-8, hi=8)
    B = synthetic.integer_matrix(K, N, seed=n + 5 * m + 7 * g, lo=-8, hi=8)
    C, C_ref, _ = _spmm(W, B, n, m, g, "f32")
    assert np.array_equal(C.cpu().numpy().astype(np.float64), C_ref)


def test_nmg_errors():
    W = torch.zeros((8, 12), device="cuda")
    with pytest.raises(sten.StenError) as e:
        sten.nmg_sparsify(W[:, :10], 2, 4, 1)                 # K = 10 not a multiple of L = 6
    assert e.value.status == 2
    W5 = torch.zeros((5, 20), device="cuda")
    v, i = sten.nmg_sparsify(W5, 2, 5, 2)                    # converts (C(5,2) = 10, L = 20)
    with pytest.raises(sten.StenError) as e:
        sten.nmg_spmm(v, i, torch.zeros((20, 8), device="cuda"), 2, 5, 2)
    assert e.value.status == 3                                # no compiled product for 2:5
    with pytest.raises(sten.StenError) as e:
        sten.nmg_sparsify(W5, 2, 5, 2, method=3)              # unknown conversion method
    assert e.value.status == 1


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n,m,g", SPMM_SET + CONVERT_ONLY)
@pytest.mark.parametrize("method", [1, 2])
def test_nmg_exchange_conversion_bit_exact(dtype, n, m, g, method):
    """The paper's GPU conversion (pattern exchange) on the GPU equals the oracle's
    sequential reading (R22) bit for bit: idx, values and densify."""
    L = oracle.nmg_chunk(n, m, g)
    M, K = 3 * m, 4 * L
    W = synthetic.weights(M, K, seed=n * 31 + m * 7 + g + method, dtype=dtype)
    v_ref, i_ref = oracle.nmg_sparsify_exchange(W, n, m, g, 0 if method == 1 else 1)
    v, i = sten.nmg_sparsify(dev(W, dtype), n, m, g, method=method)
    torch.cuda.synchronize()
    assert np.array_equal(host(i), i_ref)
    assert np.array_equal(host(v).view(np.uint8), v_ref.view(np.uint8))


@pytest.mark.parametrize("n,m,g", [(2, 4, 4), (1, 4, 4), (3, 6, 2)])
def test_nmg_exchange_integer_ties(n, m, g):
    L = oracle.nmg_chunk(n, m, g)
    W = synthetic.integer_matrix(4 * m, 4 * L, seed=n + m + g + 1, lo=-2, hi=2)
    for method in (1, 2):
        v_ref, i_ref = oracle.nmg_sparsify_exchange(W, n, m, g, 0 if method == 1 else 1)
        v, i = sten.nmg_sparsify(dev(W, "f32"), n, m, g, method=method)
        torch.cuda.synchronize()
        assert np.array_equal(host(i), i_ref) and np.array_equal(host(v), v_ref)
