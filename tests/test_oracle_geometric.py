"""Pins of the geometric-skip perturbation stream (NEXT-2; SPEC S:177's
optional mode; reading Q18) in the oracle:

  - the skip table against high-precision 1 - q^(g+1) (mpmath);
  - G(v) against its definition by brute force, and its distribution
    against the geometric law q^g p;
  - the induced distribution of gamma(t): the closed-form product and an
    enumeration of the skip process agree, sum to 1, and lie within the
    2^-32 quantisation of i.i.d. Bernoulli(p) components;
  - the oracle's trajectories against the exact stationary distribution of
    the geometric-mode matrix (long runs, 4.5 sigma), and the perturbation
    rate 1 - P(gamma = 0).
"""
import math

import mpmath
import numpy as np
import pytest

from oracle import exact, sim
from workloads import Predicate, config_model, config_predicate, model_from_lists, random_pbn


def test_table_matches_high_precision():
    mpmath.mp.dps = 40
    for n, p in [(10, 0.01), (50, 1e-4), (7, 0.3)]:
        m = random_pbn(n, 1, 2, 0, 2, p, seed=1)
        Cg = sim.geometric_table(m)
        q = 1 - mpmath.mpf(p)
        for g in range(n):
            ref = (1 - q ** (g + 1)) * 2 ** 32
            assert abs(int(Cg[g]) - float(ref)) <= 1.0 + 1e-6
        assert np.all(np.diff(Cg.astype(np.int64)) >= 0)
        assert [int(x) for x in Cg] == exact.geometric_cdf_table(m)


def test_skip_is_the_count_of_table_entries_below_the_word_and_geometric():
    m = random_pbn(12, 1, 2, 0, 2, 0.05, seed=2)
    Cg = sim.geometric_table(m)
    rng = np.random.default_rng(0)
    ws = rng.integers(0, 2 ** 32, size=200_000, dtype=np.uint64)
    for v in [0, int(Cg[0]) - 1, int(Cg[0]), int(Cg[5]), 2 ** 32 - 1] + [int(x) for x in ws[:200]]:
        assert sim.skip(Cg, v) == sum(1 for c in Cg if int(c) <= v)
    G = np.searchsorted(Cg.astype(np.uint64), ws, side="right")     # numpy's own count of entries <= v
    q = 1 - m.p
    for g in range(4):
        p_g = q ** g * m.p
        se = math.sqrt(p_g * (1 - p_g) / len(ws))
        assert abs(np.mean(G == g) - p_g) < 4.5 * se
    assert abs(np.mean(G == m.n) - q ** m.n) < 4.5 * math.sqrt(q ** m.n / len(ws))


@pytest.mark.parametrize("n,p", [(3, 0.2), (5, 0.05), (6, 0.5)])
def test_gamma_distribution_two_constructions_and_bernoulli(n, p):
    m = random_pbn(n, 1, 2, 0, 2, p, seed=3)
    A = exact.geometric_gamma_distribution(m)
    B = exact.geometric_gamma_by_enumeration(m)
    assert np.allclose(A, B, atol=1e-15, rtol=0)
    assert abs(A.sum() - 1.0) < 1e-12
    for v in range(1 << n):
        h = bin(v).count("1")
        assert abs(A[v] - p ** h * (1 - p) ** (n - h)) < 4 * n * 2.0 ** -32


def test_oracle_gamma_words_follow_the_stream_definition():
    """One chain-step by hand: the flip positions k_1 = G(v_0),
    k_{j+1} = k_j + 1 + G(v_j) from the skip words, versus the oracle's
    step (the all-constant-0 network: after a step, node i is 1 iff it was
    flipped from 0, so s_t shows gamma(t) exactly when s_{t-1} = 0)."""
    n, p = 8, 0.3
    m = model_from_lists(n, p, [[([], [0], 1.0)] for _ in range(n)])
    Cg = sim.geometric_table(m)
    pred = Predicate(np.zeros(0, np.uint16), np.zeros(0, np.uint8))
    seed = 7
    for chain in range(5):
        for t in range(1, 40):
            st, _ = sim.simulate(m, pred, seed, [chain], step0=t - 1, burn_in=0, steps=1, init=False,
                                 state=np.zeros((1, n), np.uint8), geometric=True)
            gam = np.zeros(n, np.uint8)
            k, mm = -1, 0
            while True:
                k = k + 1 + sim.skip(Cg, sim.skip_word(seed, chain, t, mm))
                mm += 1
                if k >= n:
                    break
                gam[k] = 1
            # with gamma = 0 every node applies its constant-0 function
            assert np.array_equal(st[0], gam), (chain, t)


@pytest.mark.parametrize("seed", [1, 2])
def test_geometric_mode_frequency_vs_exact(seed):
    m = random_pbn(4, 1, 3, 1, 3, 0.08, seed=20 + seed)
    pred = Predicate(np.array([0, 3], np.uint16), np.array([1, 0], np.uint8))
    T = exact.matrix_geometric(m)
    assert np.allclose(T.sum(axis=1), 1.0, atol=1e-12)
    assert np.allclose(T, exact.matrix_geometric(m, exact.geometric_gamma_by_enumeration(m)), atol=1e-15)
    pi = exact.lu_solve(T)
    target = exact.property_probability(pi, m.n, pred)
    _, I = sim.simulate(m, pred, seed=seed, chain_ids=np.arange(4), step0=0, burn_in=200, steps=100_000,
                        threads=4, geometric=True)
    bm = I.reshape(4, 50, -1).mean(axis=2).ravel()
    assert abs(bm.mean() - target) < 4.5 * bm.std(ddof=1) / math.sqrt(bm.size) + 1e-12


def test_geometric_mode_C1_vs_exact_1024_states():
    m, pred = config_model("C1"), config_predicate("C1")
    pi = exact.power_iteration(exact.matrix_geometric(m))
    target = exact.property_probability(pi, m.n, pred)
    _, I = sim.simulate(m, pred, seed=1, chain_ids=np.arange(8), step0=0, burn_in=1000, steps=100_000, threads=8,
                        geometric=True)
    bm = I.reshape(8, 50, -1).mean(axis=2).ravel()
    assert abs(bm.mean() - target) < 4.5 * bm.std(ddof=1) / math.sqrt(bm.size) + 1e-12


def test_geometric_perturbation_rate():
    """the fraction of chain-steps with gamma != 0 is 1 - P(gamma = 0)
    (all-constant-0 network from the all-zero state: I = 'all zero' is 0
    after a step iff some node was flipped)."""
    n, p = 6, 0.02
    m = model_from_lists(n, p, [[([], [0], 1.0)] for _ in range(n)])
    pred = Predicate(np.arange(n, dtype=np.uint16), np.zeros(n, np.uint8))
    _, I = sim.simulate(m, pred, seed=2, chain_ids=np.arange(4), step0=0, burn_in=1, steps=200_000, threads=4,
                        geometric=True)
    prev, nxt = I[:, :-1], I[:, 1:]
    frm = prev == 1
    rate = float(np.sum(frm & (nxt == 0))) / float(np.sum(frm))
    target = 1 - exact.geometric_gamma_distribution(m)[0]
    k = float(np.sum(frm))
    assert abs(rate - target) < 4.5 * math.sqrt(target * (1 - target) / k)
