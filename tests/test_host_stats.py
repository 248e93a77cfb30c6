"""Host-side library logic vs the oracle (no GPU): model validation, the fp64
statistics (R-hat, two-state, quantiles, Skart CI) -- 1e-9 relative
(BASELINE north_star), M and N exact unless the pre-ceil value is within
1e-9 of an integer (reading Q10, ceil tie hazard)."""
import math

import numpy as np
import pytest
import scipy.stats

import paper_1508_07828_b200 as pbn
from oracle import skart as oskart
from oracle import stats
from workloads import config_model, model_from_lists, random_pbn

REL = 1e-9


def close(a, b, rel=REL, abs_=1e-300):
    return math.isclose(a, b, rel_tol=rel, abs_tol=abs_)


def test_validate_accepts_configs():
    for k in ["C1", "C2", "C3"]:
        st, msg = pbn.pbn_validate(config_model(k))
        assert st == 0, msg


@pytest.mark.parametrize("mutate,needle", [
    ("probsum", "sum"),
    ("parent_range", "out of range"),
    ("table_len", "table"),
    ("dup_parent", "repeats parent"),
    ("p_zero", "perturbation"),
])
def test_validate_rejects(mutate, needle):
    m = random_pbn(5, 2, 2, 2, 2, 0.01, seed=3)
    if mutate == "probsum":
        m.sel_prob = m.sel_prob.copy()
        m.sel_prob[0] = 0.5
        m.sel_prob[1] = 0.4
    elif mutate == "parent_range":
        m.parents = m.parents.copy()
        m.parents[0] = 5
    elif mutate == "table_len":
        m.tbl_off = m.tbl_off.copy()
        m.tbl_off[1:] += 1
        m.tables = np.concatenate([m.tables, np.zeros(1, np.uint32)])
    elif mutate == "dup_parent":
        m.parents = m.parents.copy()
        m.parents[1] = m.parents[0]
    elif mutate == "p_zero":
        m.p = 0.0
    st, msg = pbn.pbn_validate(m)
    assert st == 1 and needle in msg, (st, msg)
    if mutate in ("probsum",):
        assert "node 0" in msg


def test_gelman_rubin_matches_oracle():
    rng = np.random.default_rng(7)
    for _ in range(200):
        omega = int(rng.integers(2, 2000))
        psi = int(rng.integers(2, 200_000))
        q = rng.random()
        c = rng.binomial(psi, q, size=omega)
        if np.all(c == 0) or np.all(c == psi):
            continue
        S1 = int(c.sum())
        S2 = int((c.astype(object) ** 2).sum())
        st, rhat, B, W, s2 = pbn.pbn_gelman_rubin(S1, S2, omega, psi)
        o = stats.gelman_rubin_counts(c, psi)
        assert st == 0
        assert close(W, o.W) and close(s2, o.sigma2) and close(rhat, o.rhat)
        assert abs(B - o.B) <= REL * max(abs(o.B), o.W * 1e-6)


def test_gelman_rubin_spec_example_and_degenerate():
    st, rhat, B, W, s2 = pbn.pbn_gelman_rubin(4, 8, 2, 4)   # windows (0101),(1010)
    assert st == 0 and B == 0 and close(W, 1 / 3, 1e-15) and close(s2, 0.25, 1e-15)
    assert close(rhat, math.sqrt(0.75), 1e-15)
    st, *_ = pbn.pbn_gelman_rubin(0, 0, 3, 10)             # all chains constant 0
    assert st == 3


def test_two_state_matches_oracle():
    rng = np.random.default_rng(11)
    for _ in range(300):
        n0 = int(rng.integers(1, 10**8))
        n1 = int(rng.integers(1, 10**8))
        n01 = int(rng.integers(0, n0 + 1))
        n10 = int(rng.integers(0, n1 + 1))
        r = float(10 ** rng.uniform(-5, -1))
        s = float(rng.uniform(0.5, 0.999))
        eps = float(10 ** rng.uniform(-12, -3))
        st, res = pbn.pbn_two_state(n01, n0, n10, n1, r, s, eps)
        o = stats.two_state(n01, n0, n10, n1, r, s, eps)
        if o.degenerate:
            assert st == 3
            continue
        assert st == 0
        assert close(res.alpha, o.alpha) and close(res.beta, o.beta)
        assert close(res.M_raw, o.M_raw) and close(res.N_raw, o.N_raw)
        if abs(o.M_raw - round(o.M_raw)) > 1e-9 * max(1, abs(o.M_raw)):
            assert res.M == o.M
        if abs(o.N_raw - round(o.N_raw)) > 1e-9 * max(1, abs(o.N_raw)):
            assert res.N == o.N


def test_two_state_spec_numbers():
    st, res = pbn.pbn_two_state(10, 100, 10, 100, 0.01, 0.95, 1e-10)
    assert st == 0 and (res.M, res.N) == (101, 86433)
    st, res = pbn.pbn_two_state(5, 10, 5, 10, 0.01, 0.95, 1e-10)
    assert st == 0 and res.M == 1
    assert pbn.pbn_two_state(0, 10, 0, 10, 0.01, 0.95, 1e-10)[0] == 3


def test_quantiles():
    for q in [1e-10, 1e-4, 0.01, 0.025, 0.2, 0.5, 0.8, 0.975, 0.999, 1 - 1e-8]:
        assert abs(pbn.pbn_inv_norm_cdf(q) - stats.inv_norm_cdf(q)) <= 1e-13 * max(1, abs(stats.inv_norm_cdf(q)))
    for df in [1, 2, 3, 5, 10, 29, 100, 1279, 10**5]:
        for q in [0.005, 0.025, 0.1, 0.5, 0.9, 0.975, 0.995]:
            ref = float(scipy.stats.t.ppf(q, df))
            got = pbn.pbn_t_quantile(q, df)
            assert abs(got - ref) <= 1e-10 * max(1.0, abs(ref)), (q, df, got, ref)
            assert abs(got - oskart.t_quantile(q, df)) <= 1e-9 * max(1.0, abs(ref))
    assert abs(pbn.pbn_t_quantile(0.975, 1) - math.tan(math.pi * 0.475)) < 1e-12


def test_skart_ci_matches_oracle():
    rng = np.random.default_rng(5)
    for _ in range(30):
        omega = int(rng.integers(1, 9))
        per = int(rng.integers(2, 200))
        kappa = int(rng.integers(1, 64))
        q = rng.uniform(0.05, 0.95)
        bs = rng.binomial(kappa, q, size=(omega, per)).astype(np.uint32)
        st, res = pbn.pbn_skart_ci_from_batches(bs, kappa, 0.05)
        o = oskart.ci_from_batches(bs, kappa, 0.05)
        assert st == 0
        for a, b in [(res.mu, o.mu), (res.var, o.var), (res.ci_lo, o.ci_lo), (res.ci_hi, o.ci_hi),
                     (res.H, o.H)]:
            assert close(a, b), (a, b)
