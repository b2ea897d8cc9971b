"""Pins of the NEXT-2 oracles (masked linear training path; fixed-mask fast
path) against what the mathematics fixes -- CPU only.

  S1 SDDMM = the dense G B^T (numpy fp64 matmul, integer inputs: exact) sampled at the kept positions
  S2 adjoint identity <densify(v) B, G> = <v, SDDMM(G, B)> (exact on integers): catches transposed
     operands, wrong index maps and dropped terms
  S3 unit perturbation: L(v + e_i) - L(v) = dV_i for the linear loss L = <densify(v) B, G>
  S4 Bound >= |dV|
  M1 mask check: W = densify(values) -> 0 outside and the values back bit-exact; one planted
     nonzero at a pruned position -> exactly 1; random W -> the count of an independent numpy mask
"""
import numpy as np
import pytest

import oracle
import synthetic

FMT = [(2, 4, 4), (1, 4, 1), (1, 10, 2), (3, 6, 3), (2, 8, 4), (1, 2, 2)]


def _setup(n, m, g, M=12, K=None, N=9, seed=0):
    K = K or 3 * m
    M = M // g * g or g
    W = synthetic.integer_matrix(M, K, seed=seed, lo=-4, hi=4)
    v, i = oracle.sparsify(W, n, m, g)
    B = synthetic.integer_matrix(K, N, seed=seed + 1, lo=-4, hi=4)
    G = synthetic.integer_matrix(M, N, seed=seed + 2, lo=-4, hi=4)
    return W, v, i, B, G


def _mask(i, n, m, g, M, K):
    """independent numpy mask of the kept positions"""
    mask = np.zeros((M, K), bool)
    for r in range(M):
        for kb in range(K // m):
            for t in range(n):
                mask[r, kb * m + int(i[r // g, kb, t])] = True
    return mask


@pytest.mark.parametrize("n,m,g", FMT)
def test_s1_sddmm_is_sampled_dense_product(n, m, g):
    W, v, i, B, G = _setup(n, m, g, seed=n + m + g)
    M, K = W.shape
    dV, _ = oracle.sddmm(G, B, i, n, m, g)
    dense = G.astype(np.float64) @ B.astype(np.float64).T          # [M][K]
    mask = _mask(i, n, m, g, M, K)
    expect = dense[mask].reshape(M, K // m * n)                      # row-major order = kept ascending
    assert np.array_equal(dV, expect)


@pytest.mark.parametrize("n,m,g", FMT)
def test_s2_adjoint_identity(n, m, g):
    W, v, i, B, G = _setup(n, m, g, seed=3 * n + m)
    C, _ = oracle.spmm(v, i, B, n, m, g)
    dV, _ = oracle.sddmm(G, B, i, n, m, g)
    assert float((C * G).sum()) == float((v.astype(np.float64) * dV).sum())


@pytest.mark.parametrize("n,m,g", FMT[:3])
def test_s3_unit_perturbation(n, m, g):
    W, v, i, B, G = _setup(n, m, g, seed=7 * n + m)
    dV, _ = oracle.sddmm(G, B, i, n, m, g)
    L0 = float((oracle.spmm(v, i, B, n, m, g)[0] * G).sum())
    rng = np.random.default_rng(1)
    for _ in range(5):
        r, kk = int(rng.integers(v.shape[0])), int(rng.integers(v.shape[1]))
        v2 = v.copy()
        v2[r, kk] += 1.0
        L1 = float((oracle.spmm(v2, i, B, n, m, g)[0] * G).sum())
        assert L1 - L0 == dV[r, kk]


@pytest.mark.parametrize("n,m,g", FMT)
def test_s4_bound(n, m, g):
    W = synthetic.weights(16 // g * g, 4 * m, seed=5)
    v, i = oracle.sparsify(W, n, m, g)
    B = synthetic.activations(4 * m, 33, seed=6)
    G = synthetic.activations(W.shape[0], 33, seed=7)
    dV, bound = oracle.sddmm(G, B, i, n, m, g)
    assert (np.abs(dV) <= bound * (1 + 1e-12)).all()


@pytest.mark.parametrize("n,m,g", FMT)
def test_m1_mask_check(n, m, g):
    W, v, i, B, G = _setup(n, m, g, seed=11 * n + m)
    M, K = W.shape
    D = oracle.densify(v, i, n, m, g, K)
    vals, out = oracle.mask_check(D, i, n, m, g)
    assert out == 0 and np.array_equal(vals, v)
    mask = _mask(i, n, m, g, M, K)
    rr, kk = np.argwhere(~mask)[0]
    D2 = D.copy()
    D2[rr, kk] = 3.0
    assert oracle.mask_check(D2, i, n, m, g)[1] == 1
    Wr = synthetic.weights(M, K, seed=9)
    Wr[np.random.default_rng(2).random((M, K)) < 0.3] = 0.0
    vals, out = oracle.mask_check(Wr, i, n, m, g)
    assert out == int(np.count_nonzero(Wr[~mask]))
    assert np.array_equal(vals, Wr[mask].reshape(M, K // m * n))
