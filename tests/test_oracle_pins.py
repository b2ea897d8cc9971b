"""Pins of the CPU oracle against things fixed OUTSIDE the oracle (-m "not gpu").

Each test names the pin from SURVEY.md 8(c) / DESIGN.md it implements:
worked examples (tests/golden, with citations), brute force over all C(m,n)
subsets, textbook per-block top-n at g = 1 (numpy lexsort), closed forms
(B = I), integer-exact products against an independent dense path and numpy,
energy inequalities from nested feasible sets, and structural invariants.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
import synthetic

NM_SET = [(1, 2), (2, 4), (1, 4), (2, 8), (1, 8), (1, 10), (1, 12), (3, 6)]


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


def _f32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float32))


def _mask_from_idx(idx, M, K, n, m, g):
    """Independent numpy scatter of the idx array into a 0/1 mask (for structure checks)."""
    mask = np.zeros((M, K), dtype=bool)
    G, KB, _ = idx.shape
    for grp in range(G):
        for kb in range(KB):
            for t in range(n):
                mask[grp * g:(grp + 1) * g, kb * m + int(idx[grp, kb, t])] = True
    return mask


# ----------------------------------------------------------------------------------------
# P0 -- hand-derived worked example (tests/golden/p0_worked_example.json)
# ----------------------------------------------------------------------------------------
def test_p0_worked_example(golden_dir):
    ex = _load(golden_dir, "p0_worked_example.json")
    n, m, g = ex["n"], ex["m"], ex["g"]
    W = _f32(ex["W"])
    values, idx = oracle.sparsify(W, n, m, g)
    assert idx.tolist() == ex["idx"]
    assert values.tolist() == ex["values"]
    B = _f32([[k + 1, 1] for k in range(W.shape[1])])
    C, Bd = oracle.spmm(values, idx, B, n, m, g)
    assert C.tolist() == ex["C"]
    Wm = oracle.densify(values, idx, n, m, g, W.shape[1])
    assert math.isclose(oracle.energy(Wm, W), ex["energy_num"] / ex["energy_den"], rel_tol=1e-15)
    v1, i1 = oracle.sparsify(W, n, m, 1)
    assert i1.tolist() == ex["g1_idx"]
    assert math.isclose(oracle.energy(oracle.densify(v1, i1, n, m, 1, W.shape[1]), W),
                        ex["g1_energy_num"] / ex["energy_den"], rel_tol=1e-15)


# ----------------------------------------------------------------------------------------
# SPEC.md worked examples (tests/golden/spec_examples.json)
# ----------------------------------------------------------------------------------------
def test_spec_examples(golden_dir):
    ex = _load(golden_dir, "spec_examples.json")
    e = ex["per_block_fraction"]
    v, i = oracle.sparsify(_f32(e["W"]), e["n"], e["m"], e["g"])
    assert i.tolist() == e["idx"] and v.tolist() == e["values"]

    e = ex["energy"]
    assert math.isclose(oracle.energy(_f32(e["Xhat"]), _f32(e["X"])), e["num"] / e["den"],
                        rel_tol=1e-15)

    e = ex["spmm_1_2_1"]
    v, i = oracle.sparsify(_f32(e["W"]), e["n"], e["m"], e["g"])
    C, _ = oracle.spmm(v, i, _f32(e["B"]), e["n"], e["m"], e["g"])
    assert C.tolist() == e["C"]

    e = ex["two_blocks_1_2_1"]
    W = _f32(e["W"])
    v, i = oracle.sparsify(W, e["n"], e["m"], e["g"])
    assert i.tolist() == e["idx"] and v.tolist() == e["values"]
    Wm = oracle.densify(v, i, e["n"], e["m"], e["g"], W.shape[1])
    assert math.isclose(oracle.energy(Wm, W), e["energy_num"] / e["energy_den"], rel_tol=1e-7)


# ----------------------------------------------------------------------------------------
# P1 -- brute force over all C(m, n) subsets on tiny integer inputs (many ties)
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("n,m", NM_SET)
@pytest.mark.parametrize("g", [1, 2, 3, 4])
def test_p1_brute_force(n, m, g):
    for seed, (lo, hi) in enumerate([(-2, 2), (-8, 8), (0, 1)]):
        W = synthetic.integer_matrix(2 * g, 3 * m, seed=100 * n + 10 * m + g + seed, lo=lo, hi=hi)
        _, idx = oracle.sparsify(W, n, m, g)
        assert np.array_equal(idx, oracle.brute_select(W, n, m, g)), (n, m, g, lo, hi)


# ----------------------------------------------------------------------------------------
# P2 -- g = 1 is textbook per-block top-n magnitude (numpy lexsort, lower index on ties)
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("n,m", NM_SET)
def test_p2_textbook_topn_g1(n, m):
    W = synthetic.weights(8, 6 * m, seed=7 + m + n)
    W[0, :m] = W[0, 0]          # an all-tied block
    W[1, :m] = -W[1, :m]        # sign must not matter
    _, idx = oracle.sparsify(W, n, m, 1)
    for r in range(W.shape[0]):
        for kb in range(W.shape[1] // m):
            a = np.abs(W[r, kb * m:(kb + 1) * m]).astype(np.float64)
            order = np.lexsort((np.arange(m), -a))     # by |w| desc, then position asc
            assert idx[r, kb].tolist() == sorted(order[:n].tolist())


# ----------------------------------------------------------------------------------------
# P3 -- crafted ties
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("n,m", NM_SET)
@pytest.mark.parametrize("g", [1, 4])
def test_p3_all_equal_and_zero_blocks(n, m, g):
    W = np.full((g, 2 * m), 0.5, np.float32)
    W[:, m:] = 0.0
    values, idx = oracle.sparsify(W, n, m, g)
    assert idx[0, 0].tolist() == list(range(n)) and idx[0, 1].tolist() == list(range(n))
    assert np.all(values[:, :n] == 0.5) and np.all(values[:, n:] == 0.0)


def test_p3_negative_zero_is_zero():
    W = _f32([[-0.0, 0.0, -0.0, 1.0]])
    _, idx = oracle.sparsify(W, 2, 4, 1)
    assert idx.tolist() == [[[0, 3]]]


# ----------------------------------------------------------------------------------------
# P4 -- energy inequalities from nested feasible sets (exact on integer inputs)
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("n,m", [(2, 4), (1, 4), (1, 8), (3, 6)])
def test_p4_energy_nesting(n, m):
    W = synthetic.integer_matrix(32, 8 * m, seed=3 * m + n, lo=-50, hi=50)
    K = W.shape[1]
    nnz = W.shape[0] * K // m * n
    a = np.sort(np.abs(W).ravel().astype(np.float64))[::-1]
    e_unstructured = a[:nnz].sum() / a.sum()
    e = {}
    for g in [1, 2, 4, 8, 16]:
        v, i = oracle.sparsify(W, n, m, g)
        e[g] = oracle.energy(oracle.densify(v, i, n, m, g, K), W)
    assert e_unstructured >= e[1]
    for g1, g2 in [(1, 2), (2, 4), (4, 8), (8, 16), (1, 16)]:
        assert e[g2] <= e[g1], (g1, g2, e)


def test_p4_energy_nesting_float_slack():
    W = synthetic.weights(64, 256, seed=11)
    e = {}
    for g in [1, 4, 16]:
        v, i = oracle.sparsify(W, 2, 4, g)
        e[g] = oracle.energy(oracle.densify(v, i, 2, 4, g, 256), W)
    assert e[4] <= e[1] * (1 + 1e-6) and e[16] <= e[4] * (1 + 1e-6)
    # sanity on the 50% point for Gaussian weights: g=1 energy of 2:4 is well above 1/2
    assert 0.5 < e[16] <= e[1] < 1.0


# ----------------------------------------------------------------------------------------
# P5 / P6 -- structure and idempotence
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("n,m", NM_SET)
@pytest.mark.parametrize("g", [1, 2, 4])
def test_p5_structure(n, m, g):
    M, K = 4 * g, 5 * m
    W = synthetic.weights(M, K, seed=m * 31 + n + g)
    values, idx = oracle.sparsify(W, n, m, g)
    assert values.shape == (M, K // m * n) and idx.shape == (M // g, K // m, n)
    assert np.all(np.diff(idx.astype(int), axis=2) > 0) if n > 1 else True
    assert idx.max() < m
    mask = _mask_from_idx(idx, M, K, n, m, g)
    assert np.all(mask.reshape(M, K // m, m).sum(axis=2) == n)
    Wm = oracle.densify(values, idx, n, m, g, K)
    assert np.array_equal(Wm.view(np.uint32), np.where(mask, W, np.float32(0)).view(np.uint32))
    # values are bit copies in ascending position order
    assert np.array_equal(values.view(np.uint32), W[mask].reshape(M, -1).view(np.uint32))
    # P6: sparsify(densify(sparsify(W))) == sparsify(W) when kept scores are > 0
    v2, i2 = oracle.sparsify(Wm, n, m, g)
    assert np.array_equal(i2, idx) and np.array_equal(v2, values)


# ----------------------------------------------------------------------------------------
# product pins: masked-dense second path, numpy, closed form B = I, exact integers
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("n,m,g", [(2, 4, 4), (1, 4, 2), (1, 10, 1), (3, 6, 3), (1, 12, 4)])
def test_spmm_integer_exact_vs_dense_paths(n, m, g):
    M, K, N = 4 * g, 6 * m, 9
    W = synthetic.integer_matrix(M, K, seed=1 + n + m + g)
    B = synthetic.integer_matrix(K, N, seed=2 + n + m + g)
    values, idx = oracle.sparsify(W, n, m, g)
    C, Bd = oracle.spmm(values, idx, B, n, m, g)
    Wm = oracle.densify(values, idx, n, m, g, K)
    assert np.array_equal(C, oracle.dense_matmul(Wm, B))
    assert np.array_equal(C, Wm.astype(np.float64) @ B.astype(np.float64))
    assert np.array_equal(Bd, np.abs(Wm).astype(np.float64) @ np.abs(B).astype(np.float64))


def test_spmm_float_vs_numpy():
    n, m, g = 2, 4, 4
    W = synthetic.weights(32, 64, seed=5)
    B = synthetic.activations(64, 40, seed=5)
    values, idx = oracle.sparsify(W, n, m, g)
    C, Bd = oracle.spmm(values, idx, B, n, m, g)
    Wm = oracle.densify(values, idx, n, m, g, 64).astype(np.float64)
    ref = Wm @ B.astype(np.float64)
    assert np.max(np.abs(C - ref) / np.maximum(Bd, 1e-300)) < 1e-14
    assert np.all(Bd >= np.abs(C))


@pytest.mark.parametrize("n,m,g", [(2, 4, 4), (1, 8, 2)])
def test_spmm_identity_is_densify(n, m, g):
    K = 4 * m
    W = synthetic.weights(2 * g, K, seed=9)
    values, idx = oracle.sparsify(W, n, m, g)
    C, _ = oracle.spmm(values, idx, np.eye(K, dtype=np.float32), n, m, g)
    assert np.array_equal(C, oracle.densify(values, idx, n, m, g, K).astype(np.float64))


def test_spmm_column_slice_matches_full():
    W = synthetic.weights(16, 32, seed=1)
    B = synthetic.activations(32, 50, seed=1)
    v, i = oracle.sparsify(W, 2, 4, 4)
    C, Bd = oracle.spmm(v, i, B, 2, 4, 4)
    Cs, Bs = oracle.spmm(v, i, B, 2, 4, 4, cols=(13, 37), nthreads=3)
    assert np.array_equal(Cs, C[:, 13:37]) and np.array_equal(Bs, Bd[:, 13:37])


# ----------------------------------------------------------------------------------------
# bf16: exact widening -- the bf16 oracle equals the fp32 oracle on the widened bytes
# ----------------------------------------------------------------------------------------
def test_bf16_widening_matches_f32():
    Wb = synthetic.weights(16, 64, seed=3, dtype="bf16")
    Bb = synthetic.activations(64, 24, seed=3, dtype="bf16")
    Wf, Bf = synthetic.bf16_bits_to_f32(Wb), synthetic.bf16_bits_to_f32(Bb)
    vb, ib = oracle.sparsify(Wb, 2, 4, 4)
    vf, i_f = oracle.sparsify(Wf, 2, 4, 4)
    assert np.array_equal(ib, i_f)
    assert np.array_equal(synthetic.bf16_bits_to_f32(vb), vf)
    assert np.array_equal(oracle.spmm(vb, ib, Bb, 2, 4, 4)[0], oracle.spmm(vf, i_f, Bf, 2, 4, 4)[0])
    Wm = oracle.densify(vb, ib, 2, 4, 4, 64)
    assert np.array_equal(synthetic.bf16_bits_to_f32(Wm), oracle.densify(vf, i_f, 2, 4, 4, 64))


def test_bf16_rounding_matches_torch():
    import torch
    x = synthetic.activations(37, 53, seed=0)
    x[0, :4] = [1.00390625, 1.01171875, -3.3895314e38, 1e-40]   # ties / large / subnormal
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(synthetic.f32_to_bf16_bits(x), ref)


def test_shape_errors():
    with pytest.raises(ValueError):
        oracle.sparsify(np.zeros((6, 8), np.float32), 2, 4, 4)     # M % g
    with pytest.raises(ValueError):
        oracle.sparsify(np.zeros((4, 10), np.float32), 2, 4, 4)    # K % m


def test_fp32_score_rounding_decides_near_ties():
    """Reading R4: scores are fp32 sums in ascending row order, RNE.
    Column 0 = 1 + 2^-24 + 2^-24: each fp32 add rounds back to 1.0 (tie to even).
    Column 1 = 1 + 2^-23 (representable).  The exact sums tie (position 0 would
    win); the fp32 scores do not (column 1 wins).  The oracle must follow fp32."""
    e = np.float32(2.0 ** -24)
    W = _f32([[1.0, 1.0], [e, 0.0], [e, 0.0]])
    _, idx = oracle.sparsify(W, 1, 2, 3)
    assert idx.tolist() == [[[0]]]
    W2 = _f32([[1.0, 1.0 + 2.0 ** -23], [e, 0.0], [e, 0.0]])
    _, idx2 = oracle.sparsify(W2, 1, 2, 3)
    assert idx2.tolist() == [[[1]]]      # exact sums: col0 = 1 + 2^-23 == col1, but fp32 col0 = 1.0


# ----------------------------------------------------------------------------------------
# NEXT-2: SameFormat re-sparsification
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("n,m,g", [(2, 4, 4), (1, 4, 1), (1, 10, 2), (3, 6, 3)])
def test_same_format_pins(n, m, g):
    W = synthetic.weights(6 * g, 5 * m, seed=n + m + g)
    v, i = oracle.sparsify(W, n, m, g)
    # on the tensor that produced the pattern, re-packing gives the sparsifier's own values
    assert np.array_equal(oracle.same_format(W, i, n, m, g), v)
    # on a new tensor W2 (e.g. after an optimizer step): densify(re-pack) = W2 masked by the OLD
    # pattern; the mask is read off the densified all-ones tensor (independent of W2)
    W2 = synthetic.weights(6 * g, 5 * m, seed=99 + n + m + g)
    v2 = oracle.same_format(W2, i, n, m, g)
    mask = oracle.densify(np.ones_like(v), i, n, m, g, W.shape[1]) != 0
    assert np.array_equal(oracle.densify(v2, i, n, m, g, W.shape[1]), np.where(mask, W2, 0).astype(np.float32))
    assert (mask.reshape(W.shape[0], -1, m).sum(axis=2) == n).all()
    # bf16 bytes are copied bit for bit
    Wb = synthetic.weights(6 * g, 5 * m, seed=7, dtype="bf16")
    vb, ib = oracle.sparsify(Wb, n, m, g)
    assert np.array_equal(oracle.same_format(Wb, ib, n, m, g), vb)


# ----------------------------------------------------------------------------------------
# NEXT-3 epilogue: GELU / bias / ReLU closed forms
# ----------------------------------------------------------------------------------------
def test_gelu_bias_act_pins():
    x = np.array([-3.0, -1.0, 0.0, 1.0, 2.5, 40.0])
    y = oracle.gelu(x)
    assert y[2] == 0.0
    assert abs(y[3] - 0.8413447460685429) < 1e-15            # GELU(1) = Phi(1)
    assert abs(y[5] - 40.0) < 1e-12                          # -> x for large x
    assert np.allclose(oracle.gelu(-x), y - x, rtol=0, atol=1e-15)   # GELU(-x) = GELU(x) - x (erf odd)
    C = np.array([[1.0, -2.0], [0.5, 0.0]])
    b = np.array([0.5, -1.0])
    assert np.array_equal(oracle.bias_act(C, b, 0), C + b[:, None])
    assert np.array_equal(oracle.bias_act(C, b, 2), np.maximum(C + b[:, None], 0))
    assert np.allclose(oracle.bias_act(C, None, 1), oracle.gelu(C))
