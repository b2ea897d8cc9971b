"""NEXT-4 (b): the Fig.-6 analogue -- kept-magnitude energy of grouped n:m (A) vs the paper's
chunked n:m:g (B) over the group size g on seeded synthetic Gaussian weights (CPU, oracle only).

PAPER.md:645-657 (section 6.1, "n:m:g structure"): the energy ||X^||_1 / ||X||_1
of n:m:g approaches plain n:m as g grows (more freedom to place each pattern).  For reading (A)
(R1) the trend is the opposite: g rows share ONE pattern per m-block, and every
g2-grouping with g1 | g2 is also a g1-grouping, so the energy can only fall with g (pin P4).

Pins (each fails on a plausible mistake in the oracle):
  * closed form: (A) at g = 1 on i.i.d. N(0, s^2) keeps in expectation the top n of m
    half-normal order statistics, E = sum_{j > m-n} E[|X|_(j)] / (m E|X|) -- computed here by
    numerical integration of the order-statistic densities (independent of the oracle);
  * (A) non-increasing in g per sample (g1 | g2 nesting; fp32 score slack 1e-6);
  * (B) increasing in g on the seed mean, by many standard errors;
  * (B) above (A) at g >= 4 and below it at g = 1 (each (B) mask is an n:m mask of the
    transposed orientation, R17, so its g = 1 energy is the most constrained);
  * (B) never above per-column top-n (N7) -- exact per sample.
"""
import math

import numpy as np
import pytest

import oracle
import synthetic

M, K = 96, 384            # divisible by every g in {1, 4, 16} and by L = C(m,n) g for the formats
SEEDS = range(100, 106)
GS = (1, 4, 16)
FORMATS = [(2, 4), (1, 4), (1, 8)]


def _energies(n, m, g):
    ea, eb, ecol = [], [], []
    for s in SEEDS:
        W = synthetic.weights(M, K, seed=s)
        v, i = oracle.sparsify(W, n, m, g)
        ea.append(oracle.energy(oracle.densify(v, i, n, m, g, K), W))
        v, i = oracle.nmg_sparsify(W, n, m, g)
        eb.append(oracle.energy(oracle.nmg_densify(v, i, n, m, g, K), W))
        # per-column top-n of every m-block of rows (the orientation of (B), R17), by numpy
        A = np.abs(W.astype(np.float64)).reshape(M // m, m, K)
        ecol.append(float(np.sort(A, axis=1)[:, m - n:, :].sum() / A.sum()))
    return np.array(ea), np.array(eb), np.array(ecol)


@pytest.fixture(scope="module")
def sweep():
    return {(n, m, g): _energies(n, m, g) for (n, m) in FORMATS for g in GS}


def _half_normal_top_n_fraction(n, m):
    """E[sum of the top n of m i.i.d. |N(0,1)|] / (m E|N(0,1)|), by quadrature of the
    order-statistic densities f_(j)(x) = m!/((j-1)!(m-j)!) F^(j-1) (1-F)^(m-j) f."""
    from scipy import integrate
    f = lambda x: math.sqrt(2 / math.pi) * math.exp(-x * x / 2)          # half-normal pdf
    F = lambda x: math.erf(x / math.sqrt(2))                             # half-normal cdf
    tot = 0.0
    for j in range(m - n + 1, m + 1):
        c = math.factorial(m) / (math.factorial(j - 1) * math.factorial(m - j))
        val, _ = integrate.quad(lambda x: x * c * F(x) ** (j - 1) * (1 - F(x)) ** (m - j) * f(x), 0, np.inf)
        tot += val
    return tot / (m * math.sqrt(2 / math.pi))


@pytest.mark.parametrize("n,m", FORMATS)
def test_grouped_g1_matches_order_statistics(sweep, n, m):
    ea, _, _ = sweep[(n, m, 1)]
    expect = _half_normal_top_n_fraction(n, m)
    # M*K/m = 9216 blocks per sample, 6 samples: the standard error is ~1e-3
    assert abs(ea.mean() - expect) < 4e-3, (ea.mean(), expect)


@pytest.mark.parametrize("n,m", FORMATS)
def test_grouped_energy_falls_with_g(sweep, n, m):
    for g1, g2 in zip(GS, GS[1:]):
        a1, a2 = sweep[(n, m, g1)][0], sweep[(n, m, g2)][0]
        assert np.all(a2 <= a1 * (1 + 1e-6)), (g1, g2, a1, a2)


@pytest.mark.parametrize("n,m", FORMATS)
def test_nmg_energy_rises_with_g(sweep, n, m):
    for g1, g2 in zip(GS, GS[1:]):
        b1, b2 = sweep[(n, m, g1)][1], sweep[(n, m, g2)][1]
        se = math.sqrt(b1.var() / len(b1) + b2.var() / len(b2))
        assert b2.mean() - b1.mean() > 5 * se, (g1, g2, b1.mean(), b2.mean(), se)


@pytest.mark.parametrize("n,m", FORMATS)
def test_nmg_vs_grouped_crossover(sweep, n, m):
    ea, eb, _ = sweep[(n, m, 1)]
    assert eb.mean() < ea.mean()
    for g in GS[1:]:
        ea, eb, _ = sweep[(n, m, g)]
        assert np.all(eb > ea), (g, ea, eb)


@pytest.mark.parametrize("n,m", FORMATS)
def test_nmg_below_per_column_top_n(sweep, n, m):
    for g in GS:
        _, eb, ecol = sweep[(n, m, g)]
        assert np.all(eb <= ecol * (1 + 1e-6)), (g, eb, ecol)
