"""Pins for the oracle's Skart pieces (PAPER Alg 2/5).

- Student-t quantile: closed forms df=1 (tan) and df=2, normal limit, mpmath;
- CI reduction identity: with zero batch-mean skewness and zero lag-1
  autocorrelation the interval is the classical mu +- t_{1-a/2,P-1} sqrt(Var/P)
  (scipy.stats.t.interval as an independent evaluator);
- batch rounding p' = omega ceil(p/omega) (1280, omega=3 -> 1281);
- von Neumann statistic: trend detected, i.i.d. accepted, and the
  classical single-chain formula;
- skewness vs scipy.stats.skew (biased moment ratio).
Skart control flow beyond these constants is "parity unpinned".
"""
import math

import mpmath
import numpy as np
import scipy.stats

from oracle import driver as odr
from oracle import skart as osk


def test_t_quantile_closed_forms():
    for q in [0.6, 0.9, 0.975, 0.995, 0.025]:
        assert abs(osk.t_quantile(q, 1) - math.tan(math.pi * (q - 0.5))) < 1e-10 * max(1, abs(math.tan(math.pi * (q - 0.5))))
        # df = 2: t = (2q - 1) / sqrt(2 q (1 - q))
        assert abs(osk.t_quantile(q, 2) - (2 * q - 1) / math.sqrt(2 * q * (1 - q))) < 1e-11
    assert abs(osk.t_quantile(0.975, 10**7) - 1.959963984540054) < 1e-6


def test_t_quantile_mpmath():
    mpmath.mp.dps = 30
    for df in [3, 17, 250]:
        for q in [0.05, 0.975]:
            f = lambda t: mpmath.betainc(mpmath.mpf(df) / 2, mpmath.mpf(1) / 2, 0,
                                         mpmath.mpf(df) / (df + t * t), regularized=True) / 2 - (
                min(q, 1 - q))
            ref = float(mpmath.findroot(f, -2))
            ref = ref if q < 0.5 else -ref
            assert abs(osk.t_quantile(q, df) - ref) < 1e-11 * max(1, abs(ref))


def test_ci_reduces_to_classical_t_interval():
    # one batch per chain -> no lag pairs (phi = 0); symmetric means -> skew = 0
    sums = np.array([[0], [4], [2], [2], [1], [3], [0], [4]], dtype=np.uint32)
    kappa = 4
    ci = osk.ci_from_batches(sums, kappa, 0.05)
    Y = sums.ravel() / kappa
    assert abs(ci.skew) < 1e-15 and ci.phi == 0.0
    lo, hi = scipy.stats.t.interval(0.95, len(Y) - 1, loc=Y.mean(), scale=Y.std(ddof=1) / math.sqrt(len(Y)))
    assert abs(ci.ci_lo - lo) < 1e-12 and abs(ci.ci_hi - hi) < 1e-12


def test_batch_rounding_spec():
    assert osk.round_batches(1280, 3) == 1281
    assert osk.round_batches(1280, 1) == 1280
    assert osk.round_batches(4096, 4096) == 4096


def test_von_neumann():
    trend = np.arange(100, dtype=np.float64)[None, :]
    assert odr.von_neumann_z(trend) > 5
    rng = np.random.default_rng(0)
    fails = sum(abs(odr.von_neumann_z(rng.normal(size=(1, 2000)))) > 4 for _ in range(50))
    assert fails == 0
    # single chain: the classical C = sum (x_{j+1}-x_j)^2 / (2 sum (x - mean)^2)
    x = rng.random(50)
    C = np.sum(np.diff(x) ** 2) / (2 * np.sum((x - x.mean()) ** 2))
    p = len(x)
    assert abs(odr.von_neumann_z(x[None, :]) - (1 - C) * math.sqrt((p * p - 1) / (p - 2))) < 1e-12
    # one mean per chain: independent chains -> pass
    assert odr.von_neumann_z(rng.random((30, 1))) == 0.0


def test_skewness_matches_scipy():
    rng = np.random.default_rng(3)
    for _ in range(5):
        x = (rng.random(1000) < rng.uniform(0.05, 0.95)).astype(np.uint8)
        assert abs(odr.skewness(x) - float(scipy.stats.skew(x))) < 1e-12
    assert math.isnan(odr.skewness(np.zeros(10)))
