"""Pins of the chunked n:m:g oracle (the paper's own format; DESIGN.md
readings R17-R21) against what the paper, SPEC.md and the mathematics fix -- CPU only.

  N1 pattern order: all C(m,n) subsets once, each ascending, adjacent patterns differ in one
     element ("differs in only one location"), starts at {0..n-1}.
  N2 SPEC.md worked examples (tests/golden/nmg_spec_examples.json).
  N3 structure: every pattern exactly g times per chunk, idx a permutation of the chunk,
     ascending inside a group, values bit-copied, densify = W (.) mask, n kept per column-block.
  N4 planted assignment: columns with one dominant pattern each (every pattern g times) are
     recovered exactly, in the stored order (pattern-major, ascending original column).
  N5 all-equal chunk: ties go to (column asc, pattern asc) -> idx = 0..L-1.
  N6 greedy <= exhaustive optimum (brute force over every valid assignment, tiny chunks).
  N7 nesting: energy(n:m:g) <= energy(per-column top-n n:m), exact on integers.
  N8 product: nmg_spmm == independent dense fp64 product on integers; B = I gives densify.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle

NMG = [(1, 2, 1), (1, 2, 3), (2, 4, 1), (2, 4, 2), (1, 4, 3), (1, 3, 2), (2, 5, 1), (1, 8, 2), (3, 6, 1)]


def golden():
    with open(os.path.join(os.path.dirname(__file__), "golden", "nmg_spec_examples.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("n,m", [(1, 2), (2, 4), (1, 4), (3, 6), (2, 5), (1, 8), (2, 8), (4, 8), (5, 10), (4, 16)])
def test_n1_revolving_door_order(n, m):
    P = oracle.nmg_patterns(n, m)
    sets = [tuple(int(x) for x in p) for p in P]
    assert sorted(sets) == list(itertools.combinations(range(m), n))      # every subset exactly once
    assert all(list(p) == sorted(p) for p in sets)
    assert sets[0] == tuple(range(n))
    for a, b in zip(sets, sets[1:]):
        assert len(set(a) & set(b)) == n - 1                              # one element out, one in


def test_n2_spec_examples():
    ex = golden()
    assert oracle.nmg_patterns(1, 2).tolist() == ex["pattern_counts"]["one_two"]
    assert len(oracle.nmg_patterns(2, 4)) == ex["pattern_counts"]["two_four_count"]
    assert len(oracle.nmg_patterns(3, 6)) == ex["pattern_counts"]["three_six_count"]
    for key in ("two_columns", "scaled_identity"):
        e = ex[key]
        W = np.array(e["W"], np.float32)
        v, i = oracle.nmg_sparsify(W, e["n"], e["m"], e["g"])
        D = oracle.nmg_densify(v, i, e["n"], e["m"], e["g"], W.shape[1])
        assert D.tolist() == e["dense"]
        assert abs(oracle.energy(D, W) - e["energy"]) < 1e-12
        assert abs(oracle.nmg_brute_best_energy(W, e["n"], e["m"], e["g"]) / np.abs(W).sum() - e["energy"]) < 1e-12


def _int_weights(M, K, seed, lo=-8, hi=8, nonzero=True):
    rng = np.random.default_rng(seed)
    W = rng.integers(lo, hi + 1, size=(M, K)).astype(np.float32)
    if nonzero:
        W[W == 0] = 1.0
    return W


@pytest.mark.parametrize("n,m,g", NMG)
def test_n3_structure(n, m, g):
    L = oracle.nmg_chunk(n, m, g)
    M, K = 3 * m, 2 * L
    W = _int_weights(M, K, seed=n + 10 * m + 100 * g)
    v, i = oracle.nmg_sparsify(W, n, m, g)
    D = oracle.nmg_densify(v, i, n, m, g, K)
    mask = D != 0                                  # W has no zeros, so the support is the mask
    assert np.array_equal(D, np.where(mask, W, 0))
    all_pats = list(itertools.combinations(range(m), n))
    for rb in range(M // m):
        blk = mask[rb * m:(rb + 1) * m]
        assert (blk.sum(axis=0) == n).all()        # n kept per column-block
        for c in range(K // L):
            ids = i[rb, c].astype(int)
            assert sorted(ids.tolist()) == list(range(L))            # permutation of the chunk
            pats = [tuple(np.nonzero(blk[:, c * L + b])[0]) for b in range(L)]
            for p in all_pats:
                assert pats.count(p) == g                             # every pattern g times
            order = oracle.nmg_patterns(n, m)
            for s in range(L):
                b = int(ids[s])
                assert pats[b] == tuple(order[s // g])                # slot s holds pattern s // g
                assert v[rb, c, s].tolist() == [W[rb * m + r, c * L + b] for r in order[s // g]]
            for p in range(len(all_pats)):
                grp = ids[p * g:(p + 1) * g]
                assert (np.diff(grp) > 0).all()                       # ascending within a group


@pytest.mark.parametrize("n,m,g", NMG)
def test_n4_planted_assignment(n, m, g):
    L = oracle.nmg_chunk(n, m, g)
    order = [tuple(p) for p in oracle.nmg_patterns(n, m)]
    rng = np.random.default_rng(7 * n + m + g)
    assign = np.repeat(np.arange(len(order)), g)
    rng.shuffle(assign)                            # column b gets pattern assign[b]
    W = np.ones((m, L), np.float32)
    for b in range(L):
        for r in order[assign[b]]:
            W[r, b] = 100.0 + b                    # dominant: any other pattern keeps <= n-1 of these
    v, i = oracle.nmg_sparsify(W, n, m, g)
    expect = [b for p in range(len(order)) for b in range(L) if assign[b] == p]
    assert i[0, 0].tolist() == expect
    assert v[0, 0, :, 0].tolist() == [100.0 + b for b in expect]


@pytest.mark.parametrize("n,m,g", NMG)
def test_n5_all_equal_ties(n, m, g):
    L = oracle.nmg_chunk(n, m, g)
    W = np.full((2 * m, 3 * L), 0.5, np.float32)
    _, i = oracle.nmg_sparsify(W, n, m, g)
    assert (i == np.arange(L, dtype=np.uint16)).all()


@pytest.mark.parametrize("n,m,g", [(1, 2, 1), (1, 2, 2), (1, 2, 3), (2, 4, 1), (1, 4, 1), (1, 3, 2), (1, 4, 2)])
@pytest.mark.parametrize("seed", range(6))
def test_n6_greedy_vs_exhaustive(n, m, g, seed):
    L = oracle.nmg_chunk(n, m, g)
    W = _int_weights(m, L, seed=seed * 31 + n + m + g, lo=-5, hi=5, nonzero=False)
    v, i = oracle.nmg_sparsify(W, n, m, g)
    got = float(np.abs(oracle.nmg_densify(v, i, n, m, g, L)).sum())
    best = oracle.nmg_brute_best_energy(W, n, m, g)
    assert got <= best + 1e-9
    # the greedy keeps at least half of the optimum: it is a greedy b-matching on a complete
    # bipartite graph (columns x pattern slots), whose weight is >= 1/2 of the maximum
    assert 2 * got >= best - 1e-9


@pytest.mark.parametrize("n,m,g", NMG)
def test_n7_nesting(n, m, g):
    L = oracle.nmg_chunk(n, m, g)
    W = _int_weights(4 * m, 3 * L, seed=n * m * g + 5, nonzero=False)
    v, i = oracle.nmg_sparsify(W, n, m, g)
    e_nmg = float(np.abs(oracle.nmg_densify(v, i, n, m, g, W.shape[1])).sum())
    A = np.abs(W.astype(np.float64)).reshape(W.shape[0] // m, m, W.shape[1])
    e_topn = float(np.sort(A, axis=1)[:, m - n:, :].sum())          # per column-block top-n
    assert e_nmg <= e_topn


@pytest.mark.parametrize("n,m,g", NMG)
def test_n8_product(n, m, g):
    L = oracle.nmg_chunk(n, m, g)
    M, K, N = 2 * m, 2 * L, 9
    W = _int_weights(M, K, seed=11 + n + m + g, nonzero=False)
    B = _int_weights(K, N, seed=13 + n + m + g, nonzero=False)
    v, i = oracle.nmg_sparsify(W, n, m, g)
    D = oracle.nmg_densify(v, i, n, m, g, K)
    C, Bound = oracle.nmg_spmm(v, i, B, n, m, g)
    assert np.array_equal(C, oracle.dense_matmul(D, B))
    assert np.array_equal(C, D.astype(np.float64) @ B.astype(np.float64))
    assert (Bound >= np.abs(C)).all()
    I = np.eye(K, dtype=np.float32)
    CI, _ = oracle.nmg_spmm(v, i, I, n, m, g)
    assert np.array_equal(CI, D.astype(np.float64))


def test_shape_errors():
    with pytest.raises(ValueError):
        oracle.nmg_sparsify(np.zeros((4, 10), np.float32), 2, 4, 1)     # K not a multiple of L = 6


# ---------------------------------------------------------------------------------------------
# X: the paper's GPU conversion by pattern exchange (R22)
#   X1 structure as N3 (every pattern g times, permutation, ascending groups, bit-copied values)
#   X2 fixed point: no pair of columns with different patterns gains by swapping (brute force over
#      every pair of the output assignment, exact integer arithmetic)
#   X3 monotone: starting from the greedy never lowers the kept L1 (exact on integers)
#   X4 <= the exhaustive optimum (tiny chunks)
#   X5 planted assignment recovered from the arbitrary start
# ---------------------------------------------------------------------------------------------
def _assignment(i_chunk, g):
    """column -> pattern id, read off the storage order (slot s holds pattern s // g)."""
    pat = np.empty(len(i_chunk), int)
    for s, b in enumerate(i_chunk.tolist()):
        pat[b] = s // g
    return pat


@pytest.mark.parametrize("n,m,g", NMG)
@pytest.mark.parametrize("init", [0, 1])
def test_x1_x2_exchange_structure_and_fixed_point(n, m, g, init):
    L = oracle.nmg_chunk(n, m, g)
    M, K = 2 * m, 2 * L
    W = _int_weights(M, K, seed=3 * n + 5 * m + 7 * g + init)
    v, i = oracle.nmg_sparsify_exchange(W, n, m, g, init)
    D = oracle.nmg_densify(v, i, n, m, g, K)
    mask = D != 0
    assert np.array_equal(D, np.where(mask, W, 0))
    order = [tuple(p) for p in oracle.nmg_patterns(n, m)]
    A = np.abs(W.astype(np.int64))
    for rb in range(M // m):
        for c in range(K // L):
            ids = i[rb, c]
            assert sorted(ids.tolist()) == list(range(L))
            pat = _assignment(ids, g)
            assert all((pat == p).sum() == g for p in range(len(order)))
            for p in range(len(order)):
                assert (np.diff(ids[p * g:(p + 1) * g].astype(int)) > 0).all()
            # magnitudes mag[b][p] (exact integers) and the 2-exchange optimality of the output
            blk = A[rb * m:(rb + 1) * m, c * L:(c + 1) * L]
            mag = np.array([[blk[list(order[p]), b].sum() for p in range(len(order))] for b in range(L)])
            for a in range(L):
                for b in range(a + 1, L):
                    pa, pb = pat[a], pat[b]
                    if pa != pb:
                        assert mag[a, pb] + mag[b, pa] <= mag[a, pa] + mag[b, pb], (a, b)


@pytest.mark.parametrize("n,m,g", NMG)
@pytest.mark.parametrize("seed", range(3))
def test_x3_exchange_never_lowers_the_greedy(n, m, g, seed):
    L = oracle.nmg_chunk(n, m, g)
    W = _int_weights(2 * m, 3 * L, seed=100 + seed, lo=-9, hi=9, nonzero=False)
    vg, ig = oracle.nmg_sparsify(W, n, m, g)
    vx, ix = oracle.nmg_sparsify_exchange(W, n, m, g, 1)
    eg = np.abs(oracle.nmg_densify(vg, ig, n, m, g, 3 * L).astype(np.float64)).sum()
    ex = np.abs(oracle.nmg_densify(vx, ix, n, m, g, 3 * L).astype(np.float64)).sum()
    assert ex >= eg


@pytest.mark.parametrize("n,m,g", [(1, 2, 1), (1, 2, 2), (1, 2, 3), (2, 4, 1), (1, 4, 1), (1, 3, 2), (1, 4, 2)])
@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("init", [0, 1])
def test_x4_exchange_vs_exhaustive(n, m, g, seed, init):
    L = oracle.nmg_chunk(n, m, g)
    W = _int_weights(m, L, seed=seed * 17 + n + m + g, lo=-5, hi=5, nonzero=False)
    v, i = oracle.nmg_sparsify_exchange(W, n, m, g, init)
    kept = np.abs(oracle.nmg_densify(v, i, n, m, g, L).astype(np.float64)).sum()
    assert kept <= oracle.nmg_brute_best_energy(W, n, m, g) + 1e-9


@pytest.mark.parametrize("n,m,g", NMG)
def test_x5_exchange_recovers_planted_assignment(n, m, g):
    L = oracle.nmg_chunk(n, m, g)
    order = [tuple(p) for p in oracle.nmg_patterns(n, m)]
    rng = np.random.default_rng(11 * n + m + 3 * g)
    assign = np.repeat(np.arange(len(order)), g)
    rng.shuffle(assign)
    W = np.ones((m, L), np.float32)
    for b in range(L):
        for r in order[assign[b]]:
            W[r, b] = 100.0 + b
    v, i = oracle.nmg_sparsify_exchange(W, n, m, g, 0)
    expect = [b for p in range(len(order)) for b in range(L) if assign[b] == p]
    assert i[0, 0].tolist() == expect
