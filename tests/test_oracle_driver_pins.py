"""Pins of the oracle's drivers (Algorithms 3, 4, 5 and the multi-property
reuse; oracle/driver.py) and of the Skart CI adjustments (oracle/skart.py)
to things other than the oracle itself:

  - the exact stationary distribution of tiny PBNs (oracle/exact.py, two
    independent matrix builders pinned in test_exact.py): the estimates of
    Algorithm 4 lie within r of the exact probability, and the Skart CI
    contains it, at the rate the methods promise;
  - a meta-state chain that is exactly a two-state Markov chain with known
    alpha = beta = p (the identity network), so alpha-hat,
    beta-hat and the estimate have closed forms;
  - an i.i.d. Bernoulli stream: the von Neumann test's
    first-attempt pass rate is the test's level (two-sided 0.20 -> 0.80);
  - re-simulation: every run's estimate, alpha-hat, beta-hat and N are
    recomputed from ONE long independent simulation of the same chains,
    sliced at the burn-in the run reports, which
    pins the driver's incremental bookkeeping (psi doubling, extend_by,
    boundary pairs, the burn-in discard, also when it runs past the sample);
  - algebra: G(t), the Skart skewness adjustment, is inverted by the cubic
    h(g) = g + 2 b g^2 + (4/3) b^2 g^3 + b (expand (1 + 2 b g)^3); the CI
    endpoints are re-derived piece by piece with independent evaluators
    (fractions for phi-hat, scipy for skewness and t quantiles);
  - brute force for the totals (A10).

Rates: fixed seeds, so every assertion is deterministic; the thresholds are
>= 3 binomial standard deviations below the nominal rate, so a correct
method passes while a plausible mistake (N or the CI half-width off by a
factor 2: coverage ~0.83) fails.
"""
import math
from fractions import Fraction

import numpy as np
import pytest
import scipy.stats

from oracle import driver as odr
from oracle import exact, sim
from oracle import skart as osk
from oracle import stats as ost
from workloads import Predicate, model_from_lists, random_pbn

PRED = Predicate(np.array([0, 1], np.uint16), np.array([1, 0], np.uint8))


def tiny_models(k=5):
    out = []
    for mi in range(k):
        m = random_pbn(8, 1, 3, 1, 3, 0.05, seed=100 + mi)
        pi = exact.lu_solve(exact.matrix_product_form(m))
        out.append((m, exact.property_probability(pi, m.n, PRED)))
    return out


# --------------------------------------------------------------------------
# Algorithm 4 and 5 against the exact steady state
# --------------------------------------------------------------------------
@pytest.mark.slow
def test_two_state_estimate_within_r_of_exact_pi():
    """omega = 4 on n <= 10 models, the estimate is within r of
    the exact probability; 5 models x 100 seeds, r = 0.01, s = 0.95."""
    hits, per_model = 0, []
    for m, target in tiny_models():
        h = 0
        for sd in range(100):
            o = odr.parallel_two_state(m, PRED, 1000 + sd, 4, 200, 1.1, 0.01, 0.95, 1e-10, 1 << 24, threads=4)
            h += abs(o.estimate - target) <= 0.01
        per_model.append(h)
        hits += h
    assert hits >= 465, per_model          # >= 93 % pooled (nominal 95 %, sd 1 %)
    assert min(per_model) >= 88, per_model


@pytest.mark.slow
def test_multi_property_estimates_within_r_of_exact_pi():
    """each of q = 3 properties estimated from one set of
    trajectories lies within r of its exact probability."""
    props = [PRED, Predicate(np.array([2], np.uint16), np.array([1], np.uint8)),
             Predicate(np.array([3, 4, 5], np.uint16), np.array([0, 1, 1], np.uint8))]
    hits = total = 0
    for mi in range(3):
        m = random_pbn(8, 1, 3, 1, 3, 0.05, seed=200 + mi)
        pi = exact.lu_solve(exact.matrix_product_form(m))
        targets = [exact.property_probability(pi, m.n, p) for p in props]
        for sd in range(50):
            o = odr.parallel_two_state_multi(m, props, 2000 + sd, 4, 200, 1.1, 0.01, 0.95, 1e-10, 1 << 24,
                                             threads=4)
            for pp, t in zip(o.per_prop, targets):
                if pp["degenerate"]:
                    continue
                total += 1
                hits += abs(pp["estimate"] - t) <= 0.01
                assert pp["N"] <= o.sample_size     # every N_p is met
    assert total >= 400
    # every property's sample is at least its own N_p, so coverage is >= nominal
    assert hits >= 0.93 * total, (hits, total)


@pytest.mark.slow
def test_skart_ci_contains_exact_pi():
    """the exact probability lies in the Skart CI; 5 models x 100
    seeds, omega = 4, H* = 0.005, alpha = 0.05."""
    hits, per_model = 0, []
    for m, target in tiny_models():
        h = 0
        for sd in range(100):
            o = odr.parallel_skart(m, PRED, 1000 + sd, 4, 200, 1.1, 0.005, 0.05, 1 << 24, threads=4)
            assert o.ci_lo <= o.estimate <= o.ci_hi
            assert max(o.estimate - o.ci_lo, o.ci_hi - o.estimate) <= 0.005    # exit rule H <= H*
            h += o.ci_lo <= target <= o.ci_hi
        per_model.append(h)
        hits += h
    assert hits >= 465, per_model
    assert min(per_model) >= 88, per_model


# --------------------------------------------------------------------------
# exactly Markov meta-state chain: the identity network
# --------------------------------------------------------------------------
def identity_network(n, p):
    """f_i(s) = s_i for every node: under VECTOR semantics node i changes
    exactly when gamma_i(t) = 1, so the indicator of "node 0 = 1" is a
    two-state Markov chain with alpha = beta = p_q (the quantised p)."""
    return model_from_lists(n, p, [[([i], [0, 1], 1.0)] for i in range(n)])


def test_identity_network_alpha_beta_equal_p():
    p = 0.02
    m = identity_network(3, p)
    pq, _ = exact.quantised_probs(m)
    pred = Predicate(np.array([0], np.uint16), np.array([1], np.uint8))
    o = odr.parallel_two_state(m, pred, 5, 8, 200, 1.1, 0.01, 0.95, 1e-10, 1 << 24, threads=4)
    # counts: alpha-hat is a binomial proportion over the 0-with-successor
    # positions; the pooled sample has ~ N / 2 of them
    se = math.sqrt(pq * (1 - pq) / (o.sample_size / 2))
    assert abs(o.alpha - pq) < 5 * se and abs(o.beta - pq) < 5 * se
    # pi(node0 = 1) = 1/2 exactly; N is sized for this accuracy
    assert abs(o.estimate - 0.5) < 0.01
    # M and N of the exact alpha = beta = p vs the run's
    a = b = pq
    M = math.log(1e-10 * (a + b) / max(a, b)) / math.log(abs(1 - a - b))
    N = a * b * (2 - a - b) / (a + b) ** 3 * ost.inv_norm_cdf(0.975) ** 2 / 0.01 ** 2
    assert abs(o.M - M) / M < 0.1 and abs(o.N - N) / N < 0.1


# --------------------------------------------------------------------------
# re-simulation pins of the drivers' bookkeeping
# --------------------------------------------------------------------------
def resimulate(model, pred, seed, omega, steps):
    _, I = sim.simulate(model, pred, seed=seed, chain_ids=np.arange(omega), step0=0, burn_in=0, steps=steps,
                        threads=4)
    return I


def pooled_counts(seqs):
    n01 = n0 = n10 = n1 = 0
    for x in seqs:
        x = np.asarray(x, np.int64)
        a, b = x[:-1], x[1:]
        n0 += int(np.sum(a == 0))
        n1 += int(np.sum(a == 1))
        n01 += int(np.sum((a == 0) & (b == 1)))
        n10 += int(np.sum((a == 1) & (b == 0)))
    return n01, n0, n10, n1


CASES = [
    # (model, pred, seed, omega, psi0, threshold, r)
    ("C1-like", random_pbn(10, 2, 2, 1, 3, 0.01, seed=1), PRED, 3, 8, 100, 1.1, 0.02),
    ("slow-2node", model_from_lists(2, 0.002, [[([0], [0, 1], 1.0)],
                                               [([0, 1], [0, 1, 1, 1], 0.9), ([], [0], 0.1)]]),
     Predicate(np.array([1], np.uint16), np.array([1], np.uint8)), 7, 4, 8, 1.5, 0.02),
    # burn-in discard longer than the sample: carried into the next extension
    ("identity-1node-carry", identity_network(1, 0.001),
     Predicate(np.array([0], np.uint16), np.array([1], np.uint8)), 3, 16, 8, 1.1, 0.1),
    ("identity-1node-multi-recheck", identity_network(1, 0.003),
     Predicate(np.array([0], np.uint16), np.array([1], np.uint8)), 3, 16, 8, 1.1, 0.05),
]


@pytest.mark.parametrize("name,model,pred,seed,omega,psi0,thr,r", CASES, ids=[c[0] for c in CASES])
def test_two_state_run_equals_long_resimulation(name, model, pred, seed, omega, psi0, thr, r):
    o = odr.parallel_two_state(model, pred, seed, omega, psi0, thr, r, 0.95, 1e-10, 1 << 24, threads=4)
    T = o.steps_per_chain
    I = resimulate(model, pred, seed, omega, T)
    start = o.psi_gr + o.discarded          # sample = s_{psi_gr + disc + 1} .. s_T
    sample = I[:, start:]
    L = T - start
    assert o.sample_size == omega * L
    assert o.estimate == pytest.approx(sample.sum() / (omega * L), rel=0, abs=1e-15)
    n01, n0, n10, n1 = pooled_counts(sample)            # no cross-chain pairs (Q7)
    assert o.alpha == pytest.approx(n01 / n0, rel=1e-15) and o.beta == pytest.approx(n10 / n1, rel=1e-15)
    ts = ost.two_state(n01, n0, n10, n1, r, 0.95, 1e-10)
    assert (o.M, o.N) == (ts.M, ts.N)
    # exit conditions of Algorithm 4: N met by the pooled sample (line 11),
    # M not larger than psi
    assert o.N <= o.sample_size and o.M <= o.psi
    # psi doubling of Algorithm 3: psi_gr = psi0 2^k, and the
    # chains ran 2 psi_gr steps before the first extension
    k = round(math.log2(o.psi_gr / psi0))
    assert o.psi_gr == psi0 * 2 ** k and o.gr_iterations == k + 1
    # the discarded prefix is M_final - psi_gr ("additional M - psi")
    assert o.discarded == (o.psi - o.psi_gr)
    if name == "identity-1node-carry":
        assert any(t[3] > t[4] for t in o.trace), "expected a discard longer than the sample"


@pytest.mark.parametrize("seed,omega", [(3, 4), (8, 5)])
def test_skart_run_equals_long_resimulation(seed, omega):
    m = random_pbn(8, 1, 3, 1, 3, 0.05, seed=101)
    o = odr.parallel_skart(m, PRED, seed, omega, 100, 1.1, 0.005, 0.05, 1 << 24, threads=4)
    kappa, p, d = o.M, o.N, o.extensions
    assert p % omega == 0 and o.sample_size == kappa * p           # Alg 5: eta = kappa p, p = ceil(p/w) w
    I = resimulate(m, PRED, seed, omega, o.steps_per_chain)
    per = p // omega
    sample = I[:, o.psi_gr:o.psi_gr + kappa * per]                 # skip the first psi of each chain (line 3)
    assert sample.shape[1] == kappa * per
    assert o.estimate == pytest.approx(sample.mean(), rel=1e-14)
    # the CI: rebuild it from the batch sums with independent evaluators
    sums = sample.reshape(omega, per, kappa).sum(axis=2)
    ci = check_ci_pieces(sums, kappa, 0.05)
    assert o.ci_lo == pytest.approx(ci[0], rel=1e-12) and o.ci_hi == pytest.approx(ci[1], rel=1e-12)
    # the last randomness test passed at spacer d, every earlier one failed
    tests = [t for t in o.trace if t[0] != "ci"]
    assert [t[4] for t in tests] == [False] * (len(tests) - 1) + [True]
    assert tests[-1][2] == d and len(tests) == d + 1


# --------------------------------------------------------------------------
# i.i.d. Bernoulli stream
# --------------------------------------------------------------------------
class BernoulliStream:
    """Sample source for the oracle drivers: omega i.i.d. Bernoulli(q) chains."""

    def __init__(self, q, omega, seed):
        self.rng = np.random.default_rng(seed)
        self.q, self.omega, self.length = q, omega, 0

    def advance(self, burn_in, steps):
        self.rng.random((self.omega, burn_in))
        self.length += burn_in + steps
        return (self.rng.random((self.omega, steps)) < self.q).astype(np.uint8)


@pytest.mark.slow
def test_skart_on_iid_bernoulli_stream():
    """Estimate within H* of q (the CI covers q at ~95 %), and the randomness
    test passes at the first attempt at its level: two-sided 0.20 -> 0.80
    (SPEC S:379 says >= 90 of 100, which the declared level 0.20 cannot give;
    DESIGN.md records the discrepancy; the mathematics pins the rate)."""
    within = first = 0
    for sd in range(100):
        src = BernoulliStream(0.3, 4, sd)
        o = odr.parallel_skart(None, None, 0, 4, 64, 1.1, 0.01, 0.05, 1 << 24, source=src)
        within += abs(o.estimate - 0.3) <= 0.01
        first += o.trace[0][4]
    assert within >= 90
    assert 68 <= first <= 92, first        # 100 x 0.8 +- 3 sd (sd = 4)


# --------------------------------------------------------------------------
# Skart CI adjustments, piece by piece
# --------------------------------------------------------------------------
def check_ci_pieces(sums, kappa, alpha):
    """Skart CI from chain-major batch sums [omega x per] of batch
    size kappa, every piece by an evaluator independent of oracle/skart.py;
    returns (lo, hi) and asserts ci_from_batches agrees with each piece."""
    sums = np.asarray(sums, np.int64)
    Y = sums / kappa
    omega, per = Y.shape
    P = Y.size
    flat = Y.ravel()
    # exact rational moments
    F = [[Fraction(int(v), kappa) for v in row] for row in sums]
    mu = sum(sum(row) for row in F) / P
    ss = sum((v - mu) ** 2 for row in F for v in row)
    lag = sum((row[k] - mu) * (row[k + 1] - mu) for row in F for k in range(per - 1))  # no cross-chain pairs (Q12)
    var = float(ss / (P - 1))
    phi = max(-0.999999, min(0.999999, float(lag / ss)))
    skew = float(scipy.stats.skew(flat, bias=True))
    A = (1 + phi) / (1 - phi)
    b = skew / (6 * math.sqrt(P))
    half = math.sqrt(A * var / P)
    tl, tu = scipy.stats.t.ppf(alpha / 2, P - 1), scipy.stats.t.ppf(1 - alpha / 2, P - 1)

    def G(t):      # the root of h(g) = t, h increasing near 0 (Newton)
        g = t
        for _ in range(100):
            h = g + 2 * b * g * g + (4 / 3) * b * b * g ** 3 + b - t
            g -= h / (1 + 4 * b * g + 4 * b * b * g * g)
        return g

    lo, hi = float(mu) + G(tl) * half, float(mu) + G(tu) * half
    ci = osk.ci_from_batches(sums.astype(np.uint32), kappa, alpha)
    assert ci.mu == pytest.approx(float(mu), rel=1e-14)
    assert ci.var == pytest.approx(var, rel=1e-12)
    assert ci.phi == pytest.approx(phi, rel=1e-10, abs=1e-14)
    assert ci.skew == pytest.approx(skew, rel=1e-10, abs=1e-13)
    assert ci.ci_lo == pytest.approx(lo, rel=1e-11) and ci.ci_hi == pytest.approx(hi, rel=1e-11)
    return lo, hi


def test_skew_adjust_inverts_willink_cubic():
    rng = np.random.default_rng(0)
    for _ in range(2000):
        b = float(rng.uniform(-0.05, 0.05))
        t = float(rng.uniform(-4, 4))
        g = osk.skew_adjust(t, b)
        assert g + 2 * b * g * g + (4 / 3) * b * b * g ** 3 + b == pytest.approx(t, abs=1e-10)
    assert osk.skew_adjust(1.7, 0.0) == 1.7


@pytest.mark.parametrize("seed", range(6))
def test_skart_ci_pieces_random_batches(seed):
    """Skewed, autocorrelated batch means (AR(1) with a skewed innovation),
    several chains: every adjustment of S:375 is exercised."""
    rng = np.random.default_rng(seed)
    omega, per = int(rng.integers(1, 5)), int(rng.integers(5, 40))
    Y = np.zeros((omega, per))
    for c in range(omega):
        x = 0.0
        for k in range(per):
            x = 0.6 * x + rng.exponential(1.0)
            Y[c, k] = x
    check_ci_pieces(np.rint(Y * 8), 8, 0.05)     # batch sums of batch size kappa = 8


def test_lag1_autocorrelation_spec_examples():
    """alternating (0,1,0,1,...) has phi-hat < 0, exact value by
    direct summation; the clamp at +-0.999999 on a long ramp."""
    Y = np.array([[0, 1, 0, 1, 0, 1, 0, 1]], np.uint32)
    ci = osk.ci_from_batches(Y, 1, 0.05)
    F = [Fraction(int(v)) for v in Y.ravel()]
    mu = sum(F) / len(F)
    exact_phi = sum((F[k] - mu) * (F[k + 1] - mu) for k in range(len(F) - 1)) / sum((v - mu) ** 2 for v in F)
    assert exact_phi < 0 and ci.phi == pytest.approx(float(exact_phi), rel=1e-15)
    # a ramp of 3e6 batch means: lag/ss = 1 - O(1/P) > 0.999999 -> clamped
    P = 3_000_000
    ramp = np.arange(P, dtype=np.uint32)[None, :]
    ci = osk.ci_from_batches(ramp, 1, 0.05)
    assert ci.phi == 0.999999


# --------------------------------------------------------------------------
# totals (A10) by brute force
# --------------------------------------------------------------------------
def test_totals_brute_force():
    rng = np.random.default_rng(4)
    for _ in range(20):
        chains = int(rng.integers(1, 9))
        W = int(rng.integers(0, 60))
        I = (rng.random((chains, W)) < rng.random()).astype(np.uint8)
        ws = [ost.window_stats(I[c], 7) for c in range(chains)]
        tot = ost.totals(ws)
        S1 = S2 = n01 = n10 = n0 = n1 = 0
        for c in range(chains):
            c1 = 0
            for t in range(W):
                c1 += int(I[c, t])
                if t + 1 < W:
                    a, b = int(I[c, t]), int(I[c, t + 1])
                    n0 += a == 0
                    n1 += a == 1
                    n01 += (a, b) == (0, 1)
                    n10 += (a, b) == (1, 0)
            S1 += c1
            S2 += c1 * c1
        assert [int(x) for x in tot] == [S1, S2, n01, n10, n0, n1]


# --------------------------------------------------------------------------
# Algorithm 3
# --------------------------------------------------------------------------
def test_gelman_rubin_stops_no_later_with_a_looser_threshold_and_window_matches_pi():
    m, target = tiny_models(1)[0]
    for seed in range(5):
        ch_a = odr.Chains(m, PRED, seed, 4, threads=4)
        ch_b = odr.Chains(m, PRED, seed, 4, threads=4)
        psi_a, rh_a, _, _ = odr.generate_converged_chains(ch_a, 128, 1.5, 1 << 24)
        psi_b, rh_b, _, win = odr.generate_converged_chains(ch_b, 128, 1.01, 1 << 24)
        assert psi_a <= psi_b and rh_a < 1.5 and rh_b < 1.01
        # the returned window is the last psi of the 2 psi simulated states
        _, I = sim.simulate(m, PRED, seed=seed, chain_ids=np.arange(4), step0=0, burn_in=0, steps=2 * psi_b,
                            threads=4)
        assert np.array_equal(win, I[:, psi_b:])
        # and the post-burn-in window estimates pi within 4.5 SE (batch means)
        bm = I[:, psi_b:].astype(float).reshape(4, 16, -1).mean(axis=2).ravel()
        assert abs(bm.mean() - target) < 4.5 * bm.std(ddof=1) / math.sqrt(bm.size) + 1e-12
