"""Oracle Skart pieces (PAPER Alg 2 / Alg 5) -- TEST
INFRASTRUCTURE ONLY.

The paper defers Skart's internals to [AJE08]; the constants and
formulas here are SPEC.md's declared defaults, see DESIGN.md
readings Q11/Q12.  Control flow beyond those constants is "parity
unpinned": oracle and library follow the same declared defaults.

Pinned pieces: Student-t quantile (closed forms df=1, df=2, normal limit,
mpmath), the t-interval reduction identity, batch rounding.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.special

from .stats import inv_norm_cdf


def t_cdf(t: float, df: float) -> float:
    """P(T <= t), Student t with df degrees of freedom, through the
    regularised incomplete beta function (library primitive)."""
    x = df / (df + t * t)
    y = (t * t) / (df + t * t)
    if x < 0.5:
        tail = 0.5 * float(scipy.special.betainc(0.5 * df, 0.5, x))
    else:   # I_x(a,b) = 1 - I_{1-x}(b,a), with 1-x formed without cancellation
        tail = 0.5 * (1.0 - float(scipy.special.betainc(0.5, 0.5 * df, y)))
    return tail if t <= 0 else 1.0 - tail


def t_quantile(q: float, df: float) -> float:
    """Bisection on the t CDF (lower half; upper half by symmetry)."""
    if not (0.0 < q < 1.0):
        raise ValueError("q must lie in (0,1)")
    if q > 0.5:
        return -t_quantile(1.0 - q, df)
    if q == 0.5:
        return 0.0
    lo, hi = -1.0, 0.0
    while t_cdf(lo, df) > q:
        lo *= 2.0
    for _ in range(400):
        mid = 0.5 * (lo + hi)
        if mid == lo or mid == hi:
            break
        if t_cdf(mid, df) < q:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


@dataclass
class SkartCI:
    mu: float
    var: float
    phi: float
    skew: float
    ci_lo: float
    ci_hi: float
    H: float
    batches: int


PHI_CLAMP = 0.999999


def skew_adjust(t: float, beta: float) -> float:
    """Skewness adjustment of a t quantile: G(t) = (cbrt(1 + 6 beta
    (t - beta)) - 1) / (2 beta), G(t) = t when beta = 0."""
    if beta == 0.0:
        return t
    return float((np.cbrt(1 + 6 * beta * (t - beta)) - 1) / (2 * beta))


def ci_from_batches(batch_sums: np.ndarray, kappa: int, alpha_conf: float) -> SkartCI:
    """Skewness- and autoregression-adjusted CI over chain-major
    batch means; lag-1 pairs never straddle chains (reading Q12)."""
    bs = np.asarray(batch_sums, dtype=np.float64)
    omega, per = bs.shape
    Y = (bs / kappa).ravel()
    P = len(Y)
    mu = float(np.sum(Y)) / P
    dev = Y - mu
    ss = float(np.sum(dev ** 2))
    if ss == 0.0:
        # all batch means equal: Var = 0, so the S:375 endpoints
        # mu + G(t) sqrt(A Var / p') are both mu (skewness 0/0 undefined,
        # reported as nan; the width does not depend on it)
        return SkartCI(mu, 0.0, 0.0, float("nan"), mu, mu, 0.0, P)
    var = ss / (P - 1)
    D = dev.reshape(omega, per)
    lag = float(np.sum(D[:, :-1] * D[:, 1:]))
    phi = lag / ss
    phi = max(-PHI_CLAMP, min(PHI_CLAMP, phi))
    skew = (float(np.sum(dev ** 3)) / P) / (ss / P) ** 1.5
    A = (1 + phi) / (1 - phi)
    beta = skew / (6.0 * math.sqrt(P))
    df = P - 1
    half = math.sqrt(A * var / P)
    lo = mu + skew_adjust(t_quantile(alpha_conf / 2, df), beta) * half
    hi = mu + skew_adjust(t_quantile(1 - alpha_conf / 2, df), beta) * half
    return SkartCI(mu, var, phi, skew, float(lo), float(hi), float(max(mu - lo, hi - mu)), P)


def round_batches(p: int, omega: int) -> int:
    """p' = omega * ceil(p / omega) (Fig. 2b)."""
    return omega * ((p + omega - 1) // omega)


def normal_limit_quantile(q: float) -> float:
    return inv_norm_cdf(q)
