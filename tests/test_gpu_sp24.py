"""GPU parity of K6, the 2:4 structured-sparse tensor-core path (NEXT-4), against the CPU oracle.

sten_sp24_pack turns (values, idx) of the grouped n:m sparsifier into the compressed 2:4
operand + metadata; sten_spmm_sp24 runs tcgen05.mma.sp.  Bars (as tests/test_gpu_parity.py):
  * B = I (P8): the product IS densify(values, idx), bit-exact -> the packing is exact;
  * integer-valued inputs (P7): bit-exact with the fp64 oracle (fp32 output);
  * Gaussian bf16 inputs: max |C - C_ref| / Bound <= 2e-2 (bf16 out) and <= 1e-5 (fp32 out,
    the products of bf16 inputs are exact in fp32 and only the fp32 accumulation rounds);
  * column sharding (P11): a token slice equals the same columns of the full product, bit for bit.
"""
import numpy as np
import pytest
import torch

import oracle
import synthetic
from paper_2304_07613_b200 import sten
from test_gpu_parity import dev, host, rel_err

pytestmark = pytest.mark.gpu

SP24_NM = [(2, 4), (1, 4), (2, 8), (1, 8), (1, 10), (1, 2), (1, 12), (2, 16), (1, 16)]


def _case(n, m, g, M, K, N, seed, integer=False):
    if integer:
        W = synthetic.integer_matrix(M, K, seed=seed, dtype="bf16")
        B = synthetic.integer_matrix(K, N, seed=seed + 1, lo=-4, hi=4, dtype="bf16")
    else:
        W = synthetic.weights(M, K, seed=seed, dtype="bf16")
        B = synthetic.activations(K, N, seed=seed, dtype="bf16")
    v, i = sten.sparsify_grouped_nm(dev(W, "bf16"), n, m, g)
    torch.cuda.synchronize()
    return W, B, v, i


def test_sp24_compatibility_rule():
    assert all(sten.sp24_compatible(n, m) for n, m in SP24_NM)
    for n, m in [(3, 6), (2, 6), (2, 10), (4, 16), (3, 4)]:
        assert not sten.sp24_compatible(n, m)
        v = torch.zeros((8, 0), dtype=torch.bfloat16, device="cuda")
        with pytest.raises(sten.StenError):
            sten.sp24_pack(v, torch.zeros((8, 0, n), dtype=torch.uint8, device="cuda"), n, m, 1, 0)


@pytest.mark.parametrize("n,m", SP24_NM)
@pytest.mark.parametrize("g", [1, 4, 16])
def test_sp24_identity_is_densify(n, m, g):
    """P8: with B = I_K the product is the dense masked weight -> every packed value and every
    metadata nibble is checked (K and M ragged against the 128-tiles)."""
    M, K = 16 * 13, m * 37 if m * 37 % 8 == 0 else m * 40
    W, _, v, i = _case(n, m, g, M, K, K, seed=3 * n + m + g)
    v24, meta = sten.sp24_pack(v, i, n, m, g, K)
    eye = torch.eye(K, dtype=torch.bfloat16, device="cuda")
    C = sten.spmm_sp24(v24, meta, M, K, eye, out_dtype=torch.float32)
    D = sten.densify(v, i, n, m, g, K)
    torch.cuda.synchronize()
    assert torch.equal(C, D.float())


@pytest.mark.parametrize("n,m", [(2, 4), (1, 4), (2, 8), (1, 10)])
@pytest.mark.parametrize("tile", [1, 2, 3, 4, 5, 6])
def test_sp24_integer_exact(n, m, tile):
    """P7: integer-valued bf16 inputs -> exact products and exact fp32 sums: bit-exact."""
    M, K, N = 300, m * 52, 333 + 3
    W, B, v, i = _case(n, m, 4, M, K, N, seed=11, integer=True)
    v_ref, i_ref = oracle.sparsify(W, n, m, 4)
    C_ref, _ = oracle.spmm(v_ref, i_ref, B, n, m, 4)
    v24, meta = sten.sp24_pack(v, i, n, m, 4, K)
    C = sten.spmm_sp24(v24, meta, M, K, dev(B, "bf16"), out_dtype=torch.float32, tile=tile)
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy().astype(np.float64), C_ref)


@pytest.mark.parametrize("n,m,g", [(2, 4, 4), (1, 4, 16), (2, 8, 1), (1, 10, 4), (1, 8, 64)])
@pytest.mark.parametrize("out", ["bf16", "f32"])
def test_sp24_gaussian_vs_oracle(n, m, g, out):
    M, K, N = 512, 1024 if m != 10 else 1000, 640
    W, B, v, i = _case(n, m, g, M, K, N, seed=21)
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    C_ref, Bound = oracle.spmm(v_ref, i_ref, B, n, m, g)
    assert np.array_equal(host(i), i_ref)
    v24, meta = sten.sp24_pack(v, i, n, m, g, K)
    C = sten.spmm_sp24(v24, meta, M, K, dev(B, "bf16"),
                       out_dtype=torch.float32 if out == "f32" else torch.bfloat16)
    torch.cuda.synchronize()
    e = rel_err(C, C_ref, Bound)
    assert e <= (1e-5 if out == "f32" else 2e-2), e


def test_sp24_column_shards_bit_exact():
    """P11: columns are independent and the k order does not depend on the token tiling."""
    n, m, g, M, K, N = 2, 4, 4, 384, 768, 1024
    W, B, v, i = _case(n, m, g, M, K, N, seed=5)
    v24, meta = sten.sp24_pack(v, i, n, m, g, K)
    Bd = dev(B, "bf16")
    C = sten.spmm_sp24(v24, meta, M, K, Bd, out_dtype=torch.float32)
    for c0, c1 in [(0, 256), (256, 640), (640, 1024)]:
        Cs = sten.spmm_sp24(v24, meta, M, K, Bd[:, c0:c1], out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert torch.equal(Cs, C[:, c0:c1])


def test_sp24_bench_size_sampled():
    """C3 shape at full size (BERT-large FFN, 1:4, g = 4, 16384 tokens) on sampled columns."""
    n, m, g, M, K, N = 1, 4, 4, 1024, 4096, 16384
    W, B, v, i = _case(n, m, g, M, K, N, seed=1236)
    v24, meta = sten.sp24_pack(v, i, n, m, g, K)
    C = sten.spmm_sp24(v24, meta, M, K, dev(B, "bf16"))
    torch.cuda.synchronize()
    cols = np.r_[0:64, 8000:8064, N - 64:N]
    v_ref, i_ref = oracle.sparsify(W, n, m, g)
    C_ref, Bound = oracle.spmm(v_ref, i_ref, np.ascontiguousarray(B[:, cols]), n, m, g)
    e = rel_err(C[:, torch.from_numpy(cols).cuda()], C_ref, Bound)
    assert e <= 2e-2, e
