"""Oracle statistics, fp64, written from PAPER.md and computed BY DEFINITION.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Everything here works from the stored 0/1 indicator sequences (or, where
only per-chain counts exist, from the multiset of 0/1 values a count
determines) with plain numpy / Python arithmetic in the paper's order.
Nothing here is shared with the product's C++ statistics.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


# --------------------------------------------------------------------------
# Per-chain window statistics (PAPER P:428-429, P:488,
# Fig. 2).  I is one chain's recorded window, I[0] the earliest.
# --------------------------------------------------------------------------
@dataclass
class WindowStats:
    c1: int            # number of elements equal to 1 (meta state 1)
    n01: int           # pairs (I[t-1], I[t]) = (0, 1) inside the window
    n10: int           # pairs (1, 0) inside the window
    n0from: int        # positions t < W-1 with I[t] = 0 (0-with-successor)
    n1from: int        # positions t < W-1 with I[t] = 1
    first: int
    last: int
    batch_sums: np.ndarray   # sums of consecutive batch-sized blocks from the start
    bits: np.ndarray         # packed uint32, bit t%32 of word t//32 = I[t]


def window_stats(I: np.ndarray, batch: int) -> WindowStats:
    I = np.asarray(I, dtype=np.int64)
    W = len(I)
    c1 = int(I.sum())
    prev, nxt = I[:-1], I[1:]
    n01 = int(np.sum((prev == 0) & (nxt == 1)))
    n10 = int(np.sum((prev == 1) & (nxt == 0)))
    n0from = int(np.sum(prev == 0))
    n1from = int(np.sum(prev == 1))
    first = int(I[0]) if W else 0
    last = int(I[-1]) if W else 0
    nb = (W + batch - 1) // batch if batch > 0 else 0
    batch_sums = np.array([int(I[b * batch:(b + 1) * batch].sum()) for b in range(nb)],
                          dtype=np.int64)
    nw = (W + 31) // 32
    bits = np.zeros(nw, dtype=np.uint32)
    for t in np.nonzero(I)[0]:
        bits[t // 32] |= np.uint32(1) << np.uint32(t % 32)
    return WindowStats(c1, n01, n10, n0from, n1from, first, last, batch_sums, bits)


def totals(stats: list[WindowStats]) -> np.ndarray:
    """(S1, S2, sum n01, sum n10, sum n0from, sum n1from) as exact integers."""
    S1 = sum(s.c1 for s in stats)
    S2 = sum(s.c1 * s.c1 for s in stats)
    return np.array([S1, S2, sum(s.n01 for s in stats), sum(s.n10 for s in stats),
                     sum(s.n0from for s in stats), sum(s.n1from for s in stats)],
                    dtype=np.uint64)


# --------------------------------------------------------------------------
# Gelman & Rubin, Algorithm 3, two-pass per chain.
# --------------------------------------------------------------------------
@dataclass
class Psrf:
    B: float
    W: float
    sigma2: float
    rhat: float


def _psrf_from_moments(mu_i: np.ndarray, s2_i: np.ndarray, psi: int) -> Psrf:
    omega = len(mu_i)
    mu = float(np.sum(mu_i)) / omega
    B = psi / (omega - 1) * float(np.sum((mu_i - mu) ** 2))
    W = float(np.sum(s2_i)) / omega
    sigma2 = (1.0 - 1.0 / psi) * W + B / psi
    rhat = math.sqrt(sigma2 / W) if W > 0 else float("nan")
    return Psrf(B, W, sigma2, rhat)


def gelman_rubin_windows(windows: np.ndarray) -> Psrf:
    """windows: omega x psi array of the last psi values of each chain."""
    omega, psi = np.shape(windows)
    if omega < 2 or psi < 2:
        raise ValueError("need omega >= 2 and psi >= 2")
    mu_i = np.zeros(omega)
    s2_i = np.zeros(omega)
    for i in range(omega):                   # one chain at a time (large windows stay small in memory)
        x = np.asarray(windows[i], dtype=np.float64)
        mu_i[i] = x.mean()
        s2_i[i] = ((x - mu_i[i]) ** 2).sum() / (psi - 1)               # P:429 (divisor psi-1)
    return _psrf_from_moments(mu_i, s2_i, psi)


def gelman_rubin_counts(c: np.ndarray, psi: int) -> Psrf:
    """Same statistic when each chain's window is known by its count c_i of
    ones: the window is the multiset {1 x c_i, 0 x (psi - c_i)}, so the
    two-pass moments are taken over that multiset."""
    c = np.asarray(c, dtype=np.float64)
    omega = len(c)
    if omega < 2 or psi < 2:
        raise ValueError("need omega >= 2 and psi >= 2")
    mu_i = c / psi
    s2_i = (c * (1.0 - mu_i) ** 2 + (psi - c) * (0.0 - mu_i) ** 2) / (psi - 1)
    return _psrf_from_moments(mu_i, s2_i, psi)


# --------------------------------------------------------------------------
# Normal quantile: bisection on Phi(x) = erfc(-x/sqrt 2)/2 (libm erfc is the
# primitive).  Plain and slow on purpose.
# --------------------------------------------------------------------------
def norm_cdf(x: float) -> float:
    return 0.5 * math.erfc(-x / math.sqrt(2.0))


def inv_norm_cdf(q: float) -> float:
    if not (0.0 < q < 1.0):
        raise ValueError("q must lie in (0,1)")
    if q > 0.5:
        # symmetry Phi^-1(q) = -Phi^-1(1-q); 1-q is exact for q in (0.5, 1)
        return -inv_norm_cdf(1.0 - q)
    lo, hi = -40.0, 0.0
    for _ in range(300):
        mid = 0.5 * (lo + hi)
        if mid == lo or mid == hi:
            break
        if norm_cdf(mid) < q:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


# --------------------------------------------------------------------------
# Two-state Markov chain approach, Algorithm 1 line 8.
# --------------------------------------------------------------------------
@dataclass
class TwoState:
    alpha: float
    beta: float
    M_raw: float
    N_raw: float
    M: int
    N: int
    degenerate: bool


def estimate_alpha_beta(seqs: list[np.ndarray]) -> tuple[int, int, int, int]:
    """Pooled transition counts over several 0/1 sequences; pairs are
    counted only inside each sequence (reading Q7).  Returns
    (n01, n0from, n10, n1from)."""
    n01 = n0 = n10 = n1 = 0
    for s in seqs:
        s = np.asarray(s, dtype=np.int64)
        a, b = s[:-1], s[1:]                   # the pairs (I[t-1], I[t]) of this sequence
        n0 += int(np.sum(a == 0))
        n1 += int(np.sum(a == 1))
        n01 += int(np.sum((a == 0) & (b == 1)))
        n10 += int(np.sum((a == 1) & (b == 0)))
    return n01, n0, n10, n1


def two_state(n01: int, n0from: int, n10: int, n1from: int, r: float, s: float,
              eps: float) -> TwoState:
    if n0from == 0 or n1from == 0:
        return TwoState(float("nan"), float("nan"), float("nan"), float("nan"), 0, 0, True)
    alpha = n01 / n0from                      # 0 -> 1
    beta = n10 / n1from                       # 1 -> 0
    apb = alpha + beta
    if apb == 0.0 or apb == 2.0:
        return TwoState(alpha, beta, float("nan"), float("nan"), 0, 0, True)
    # M := ceil( log( eps (alpha+beta) / max(alpha,beta) ) / log |1 - alpha - beta| )
    if abs(1.0 - apb) == 0.0:
        M_raw = 1.0                            # instant mixing (reading Q10)
    else:
        M_raw = math.log(eps * apb / max(alpha, beta)) / math.log(abs(1.0 - apb))
    z = inv_norm_cdf(0.5 * (1.0 + s))
    # N := ceil( alpha beta (2 - alpha - beta) / (alpha+beta)^3 * (Phi^-1((1+s)/2))^2 / r^2 )
    N_raw = alpha * beta * (2.0 - apb) / apb ** 3 * z * z / (r * r)
    return TwoState(alpha, beta, M_raw, N_raw, int(math.ceil(M_raw)), int(math.ceil(N_raw)),
                    False)
