"""Pins for oracle/stats.py.

- window statistics vs pure-Python brute force on tiny sequences and the
  invariants n01 - n10 = last - first, sum(batches) = c1, popcount = c1;
- Gelman & Rubin worked example (B=0, W=1/3, sigma2=1/4,
  R-hat=sqrt(3/4)); identical chains R-hat = sqrt(1-1/psi) (closed form);
- two-state worked numbers M=101, N=86433 for alpha=beta=0.1 (SPEC
  S:298; high-precision values 100.0822... and 86432.82...);
  alpha/beta examples S:289-291;
- Phi^-1 vs scipy.special.ndtri and mpmath.
"""
import math

import mpmath
import numpy as np
import pytest
import scipy.special

from oracle import stats


def brute_window(I, batch):
    W = len(I)
    c1 = 0
    n01 = n10 = n0 = n1 = 0
    for t in range(W):
        c1 += I[t]
        if t + 1 < W:
            if I[t] == 0:
                n0 += 1
                if I[t + 1] == 1:
                    n01 += 1
            else:
                n1 += 1
                if I[t + 1] == 0:
                    n10 += 1
    sums = []
    b = 0
    while b * batch < W:
        sums.append(sum(I[b * batch:(b + 1) * batch]))
        b += 1
    return c1, n01, n10, n0, n1, sums


@pytest.mark.parametrize("seed", range(20))
def test_window_stats_brute_force(seed):
    rng = np.random.default_rng(seed)
    W = int(rng.integers(1, 200))
    I = (rng.random(W) < rng.random()).astype(np.uint8)
    batch = int(rng.integers(1, 40))
    ws = stats.window_stats(I, batch)
    c1, n01, n10, n0, n1, sums = brute_window([int(x) for x in I], batch)
    assert (ws.c1, ws.n01, ws.n10, ws.n0from, ws.n1from) == (c1, n01, n10, n0, n1)
    assert list(ws.batch_sums) == sums
    assert ws.n01 - ws.n10 == ws.last - ws.first
    assert int(ws.batch_sums.sum()) == ws.c1
    assert sum(bin(int(w)).count("1") for w in ws.bits) == ws.c1
    for t in range(W):
        assert ((int(ws.bits[t // 32]) >> (t % 32)) & 1) == I[t]


def test_gelman_rubin_spec_example():
    g = stats.gelman_rubin_windows(np.array([[0, 1, 0, 1], [1, 0, 1, 0]]))
    assert g.B == 0.0
    assert math.isclose(g.W, 1 / 3, rel_tol=1e-15)
    assert math.isclose(g.sigma2, 0.25, rel_tol=1e-15)
    assert math.isclose(g.rhat, math.sqrt(0.75), rel_tol=1e-15)
    g2 = stats.gelman_rubin_counts(np.array([2, 2]), 4)
    assert (g2.B, g2.rhat) == (0.0, g.rhat)


def test_gelman_rubin_identical_chains_closed_form():
    rng = np.random.default_rng(0)
    for psi in [4, 17, 1000]:
        row = (rng.random(psi) < 0.3).astype(np.uint8)
        if row.sum() in (0, psi):
            row[0] ^= 1
        g = stats.gelman_rubin_windows(np.stack([row] * 5))
        assert g.B == 0.0
        assert math.isclose(g.rhat, math.sqrt(1 - 1 / psi), rel_tol=1e-14)


def test_gelman_rubin_counts_equals_windows():
    rng = np.random.default_rng(3)
    for _ in range(20):
        omega, psi = int(rng.integers(2, 30)), int(rng.integers(2, 300))
        X = (rng.random((omega, psi)) < rng.random()).astype(np.uint8)
        a = stats.gelman_rubin_windows(X)
        b = stats.gelman_rubin_counts(X.sum(axis=1), psi)
        for x, y in [(a.B, b.B), (a.W, b.W), (a.sigma2, b.sigma2)]:
            assert math.isclose(x, y, rel_tol=1e-12, abs_tol=1e-300)
        # sigma2 is a convex combination of W and B
        assert min(a.W, a.B) - 1e-15 <= a.sigma2 <= max(a.W, a.B) + 1e-15


def test_two_state_spec_numbers():
    # alpha = beta = 0.1 as exact counts
    ts = stats.two_state(10, 100, 10, 100, r=0.01, s=0.95, eps=1e-10)
    assert (ts.M, ts.N) == (101, 86433)
    # high-precision evaluation of the same formulas (mpmath, 40 digits)
    mpmath.mp.dps = 40
    a = mpmath.mpf("0.1")
    M_hp = mpmath.log(mpmath.mpf("1e-10") * 2 * a / a) / mpmath.log(1 - 2 * a)
    z = mpmath.sqrt(2) * mpmath.erfinv(mpmath.mpf("0.95"))
    N_hp = a * a * (2 - 2 * a) / (2 * a) ** 3 * z**2 / mpmath.mpf("0.01") ** 2
    assert abs(ts.M_raw - float(M_hp)) < 1e-10
    assert abs(ts.N_raw - float(N_hp)) < 1e-6


def test_alpha_beta_spec_examples():
    assert stats.estimate_alpha_beta([np.array([0, 0, 1, 1, 0])]) == (1, 2, 1, 2)
    n01, n0, n10, n1 = stats.estimate_alpha_beta([np.array([0, 1, 0, 1, 0, 1])])
    assert (n01 / n0, n10 / n1) == (1.0, 1.0)
    ts = stats.two_state(0, 3, 0, 0, 0.01, 0.95, 1e-10)
    assert ts.degenerate
    # no cross-chain pairs (reading Q7): [0,1] + [0,1] has two 0->1 pairs, not a 1->0
    assert stats.estimate_alpha_beta([np.array([0, 1]), np.array([0, 1])]) == (2, 2, 0, 0)


def test_two_state_singular_branches():
    assert stats.two_state(5, 10, 5, 10, 0.01, 0.95, 1e-10).M == 1     # alpha+beta = 1
    assert stats.two_state(0, 10, 0, 10, 0.01, 0.95, 1e-10).degenerate  # alpha+beta = 0
    assert stats.two_state(10, 10, 10, 10, 0.01, 0.95, 1e-10).degenerate  # periodic


def test_inv_norm_cdf_vs_scipy_and_mpmath():
    mpmath.mp.dps = 40
    qs = [1e-12, 1e-6, 0.001, 0.025, 0.1, 0.3, 0.5, 0.7, 0.9, 0.975, 0.995, 1 - 1e-9]
    for q in qs:
        x = stats.inv_norm_cdf(q)
        ref = float(mpmath.sqrt(2) * mpmath.erfinv(2 * mpmath.mpf(q) - 1))
        assert abs(x - ref) <= 1e-13 * max(1.0, abs(ref)), (q, x, ref)
        assert abs(x - float(scipy.special.ndtri(q))) <= 1e-12 * max(1.0, abs(ref))
    assert abs(stats.inv_norm_cdf(0.5)) < 1e-15
    for q in [0.01, 0.2, 0.45]:                     # symmetry q vs 1-q
        assert abs(stats.inv_norm_cdf(q) + stats.inv_norm_cdf(1 - q)) < 1e-12
    assert abs(stats.inv_norm_cdf(0.975) - 1.959963984540054) < 1e-14
