"""Oracle drivers: Algorithms 3, 4 and 5 of PAPER.md over the oracle simulator.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Every decision is taken from the stored 0/1 indicator sequences of each
chain by definition (oracle/stats.py, oracle/skart.py); nothing is shared
with the product's C++ driver.  Readings: Q7 boundary pairs,
Q8 Gelman-Rubin details, Q9 Algorithm 4 garbles, Q11/Q12 Skart constants.

Chain bookkeeping: `seq[c]` holds the indicator of chain c for every state
after the Gelman-Rubin burn-in, i.e. states s_{psi+1}, s_{psi+2}, ... of the
final GR length 2 psi (the GR window first, then every extension).

Sample source: by default the oracle simulator (`Chains`).  Any object with
the same two members -- `length` (transitions simulated per chain) and
`advance(burn_in, steps) -> I [omega x steps]` (the indicator of the
recorded states) -- can stand in for it, e.g. an i.i.d. Bernoulli stream in
the Skart pins.  The decisions below only ever look at the
indicator sequences the source returns.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import sim
from . import skart as osk
from . import stats as ost


@dataclass
class RunResult:
    estimate: float
    rhat: float
    psi: int
    steps_per_chain: int
    gr_iterations: int
    extensions: int = 0
    sample_size: int = 0
    M: int = 0
    N: int = 0
    alpha: float = float("nan")
    beta: float = float("nan")
    ci_lo: float = float("nan")
    ci_hi: float = float("nan")
    psi_gr: int = 0          # psi returned by Algorithm 3: the sample starts at state s_{psi_gr+1}
    discarded: int = 0       # elements dropped at the front of every chain's sample (Alg 4 re-check)
    trace: list = field(default_factory=list)


class Chains:
    """omega oracle chains advanced together; keeps each chain's indicator
    history from a given start and its current state."""

    def __init__(self, model, pred, seed: int, omega: int, threads: int = 8):
        self.model, self.pred, self.seed, self.omega = model, pred, seed, omega
        self.ids = np.arange(omega, dtype=np.uint32)
        self.state = None
        self.length = 0          # transitions simulated per chain
        self.threads = threads

    def advance(self, burn_in: int, steps: int) -> np.ndarray:
        """Simulate burn_in + steps transitions; returns I [omega x steps]."""
        init = self.state is None
        st, I = sim.simulate(self.model, self.pred, self.seed, self.ids, self.length, burn_in, steps,
                             init=init, state=self.state, threads=self.threads)
        self.state = st
        self.length += burn_in + steps
        return I


def generate_converged_chains(ch: Chains, psi0: int, threshold: float, max_steps: int):
    """Algorithm 3.  Returns (psi, rhat, iterations, window
    [omega x psi] = the last psi indicators of each chain) or raises."""
    psi = psi0
    window = ch.advance(psi, psi)          # trajectories of length 2 psi; last psi recorded
    it = 0
    while True:
        it += 1
        varying = np.any(window.min(axis=1) != window.max(axis=1))    # some window not constant
        g = ost.gelman_rubin_windows(window) if varying else None
        rhat = g.rhat if g is not None else float("nan")
        if g is not None and rhat < threshold:
            return psi, rhat, it, window
        if 4 * psi > max_steps:
            raise RuntimeError("Gelman-Rubin did not converge within the step cap")
        psi *= 2
        window = ch.advance(0, psi)        # extend to 2 psi: the new window is the new segment


def parallel_two_state(model, pred, seed: int, omega: int, psi0: int, threshold: float, r: float,
                       s: float, eps: float, max_steps: int, threads: int = 8, source=None) -> RunResult:
    """Algorithm 4 with reading Q9: extend by ceil((N - omega n)/omega)
    while N > omega n; then if M > psi discard M - psi more initial elements of
    every chain's sample, set psi := M and re-enter; stop when M <= psi.

    "additional M - psi elements will be discarded in the beginning of each
    chain": when that is more than the current sample holds, the
    sample is empty and the discard continues into the next extension (the
    discarded prefix is never shortened)."""
    ch = source if source is not None else Chains(model, pred, seed, omega, threads)
    psi, rhat, it, window = generate_converged_chains(ch, psi0, threshold, max_steps)
    psi_gr = psi
    seq = np.array(window, dtype=np.uint8)           # [omega x length] per-chain sample (GR window first)
    disc = 0                                         # elements discarded at the front
    ext_count = 0
    trace = []
    while True:
        while True:
            L = max(seq.shape[1] - disc, 0)
            counts = ost.estimate_alpha_beta(list(seq[:, disc:])) if L >= 2 else None
            ts = ost.two_state(*counts, r, s, eps) if counts is not None else None
            if ts is not None and not ts.degenerate:
                if ts.N <= omega * L:
                    break
                ext = -(-(ts.N - omega * L) // omega)
            else:
                ext = max(L, psi)
            if ch.length + ext > max_steps:
                raise RuntimeError("two-state sample exceeds the step cap")
            I = ch.advance(0, ext)
            seq = np.concatenate([seq, np.asarray(I, np.uint8)], axis=1)
            ext_count += 1
        if ts.M > psi:
            disc += ts.M - psi
            trace.append(("recheck", ts.M, psi, disc, seq.shape[1]))
            psi = ts.M
            continue
        break
    L = seq.shape[1] - disc
    total_ones = int(seq[:, disc:].sum(dtype=np.int64))
    return RunResult(estimate=total_ones / (omega * L), rhat=rhat, psi=psi, steps_per_chain=ch.length,
                     gr_iterations=it, extensions=ext_count, sample_size=omega * L, M=ts.M, N=ts.N,
                     alpha=ts.alpha, beta=ts.beta, psi_gr=psi_gr, discarded=disc, trace=trace)


# --------------------------------------------------------------------------
# Algorithm 4 with the multi-property reuse of samples (reading Q13)
# --------------------------------------------------------------------------
@dataclass
class MultiResult:
    rhat: float
    psi: int
    steps_per_chain: int
    gr_iterations: int
    extensions: int
    sample_size: int
    per_prop: list          # per property: dict(estimate, M, N, alpha, beta, degenerate)


def parallel_two_state_multi(model, preds, seed: int, omega: int, psi0: int, threshold: float, r: float,
                             s: float, eps: float, max_steps: int, threads: int = 8,
                             sources=None) -> MultiResult:
    """q properties checked on one set of omega trajectories.

    "The simulated samples are abstracted into different meta states based on
    these different q properties simultaneously": one oracle
    chain set per property, all with the same seed and chain ids, hence the
    same trajectories.  Gelman & Rubin: converged when every property with
    non-constant windows has R-hat < threshold (Q8).  "The next extension
    length is determined by the minimal value of all the calculated Ns"
    (P:521): grow the pooled sample to the smallest N_p not yet met, then
    re-evaluate; stop "when all the calculated Ns are smaller than the
    current sample size".  Degenerate properties are reported and do
    not drive the extension.  Burn-in re-check with the largest
    M_p (reading Q9)."""
    q = len(preds)
    chs = sources if sources is not None else [Chains(model, pr, seed, omega, threads) for pr in preds]
    psi = psi0
    windows = [ch.advance(psi, psi) for ch in chs]
    it = 0
    while True:
        it += 1
        rh = []
        for w in windows:
            if np.any(w.min(axis=1) != w.max(axis=1)):
                rh.append(ost.gelman_rubin_windows(w).rhat)
        if rh and all(x < threshold for x in rh):
            rhat = max(rh)
            break
        if 4 * psi > max_steps:
            raise RuntimeError("Gelman-Rubin did not converge within the step cap")
        psi *= 2
        windows = [ch.advance(0, psi) for ch in chs]
    seqs = [np.array(w, dtype=np.uint8) for w in windows]      # per property [omega x length]
    disc, ext_count = 0, 0
    while True:
        while True:
            L = max(seqs[0].shape[1] - disc, 0)
            ts = []
            for p in range(q):
                counts = ost.estimate_alpha_beta(list(seqs[p][:, disc:])) if L >= 2 else None
                t = ost.two_state(*counts, r, s, eps) if counts is not None else None
                ts.append(t if (t is not None and not t.degenerate) else None)
            usable = [t for t in ts if t is not None]
            if usable:
                unmet = [t.N for t in usable if t.N > omega * L]
                if not unmet:
                    break
                ext = -(-(min(unmet) - omega * L) // omega)
            else:
                ext = max(L, psi)
            if chs[0].length + ext > max_steps:
                raise RuntimeError("two-state sample exceeds the step cap")
            for p in range(q):
                I = chs[p].advance(0, ext)
                seqs[p] = np.concatenate([seqs[p], np.asarray(I, np.uint8)], axis=1)
            ext_count += 1
        Mmax = max([t.M for t in ts if t is not None], default=0)
        if Mmax > psi:
            disc += Mmax - psi
            psi = Mmax
            continue
        break
    L = seqs[0].shape[1] - disc
    per = []
    for p in range(q):
        ones = int(seqs[p][:, disc:].sum(dtype=np.int64))
        t = ts[p]
        per.append({"estimate": ones / (omega * L), "degenerate": t is None,
                    "M": t.M if t else 0, "N": t.N if t else 0,
                    "alpha": t.alpha if t else float("nan"), "beta": t.beta if t else float("nan")})
    return MultiResult(rhat=rhat, psi=psi, steps_per_chain=chs[0].length, gr_iterations=it,
                       extensions=ext_count, sample_size=omega * L, per_prop=per)


# --------------------------------------------------------------------------
# Algorithm 5 (parallel Skart), constants of SPEC S:375 (reading Q11/Q12)
# --------------------------------------------------------------------------
SKEW_LIMIT = 4.0          # |B| <= 4 -> kappa = 1, else 16
RANDOMNESS_LEVEL = 0.20   # von Neumann test, two-sided
P_CEILING = 1024          # batch-count growth ceiling in the CI loop
MAX_SKART_ITERS = 64


def skewness(x: np.ndarray) -> float:
    x = np.asarray(x, dtype=np.float64)
    m = x.mean()
    m2 = float(np.mean((x - m) ** 2))
    if m2 == 0.0:
        return float("nan")
    return float(np.mean((x - m) ** 3)) / m2 ** 1.5


def von_neumann_z(means: np.ndarray) -> float:
    """Randomness statistic over per-chain sequences of batch means (SPEC
    S:240) with successive differences taken only inside chains (reading
    Q12): C = (mean squared successive difference over the m-1 within-chain
    pairs) / (2 x sample variance of all means), z = (1-C) sqrt((m^2-1)/(m-2))
    with m = pairs + 1.  For one chain this is the classical statistic.
    Returns 0 (a pass) when there are fewer than 2 within-chain pairs: batch
    means of different converged chains are independent."""
    Y = np.asarray(means, dtype=np.float64)         # omega x k
    omega, k = Y.shape
    pairs = omega * (k - 1)
    if pairs < 2:
        return 0.0
    flat = Y.ravel()
    P = flat.size
    mu = float(np.sum(flat)) / P
    ss = float(np.sum((flat - mu) ** 2))
    if ss == 0.0:
        return float("inf")
    msd = float(np.sum((Y[:, 1:] - Y[:, :-1]) ** 2)) / pairs
    Cst = msd / (2.0 * ss / (P - 1))
    m = pairs + 1
    return (1.0 - Cst) * math.sqrt((m * m - 1.0) / (m - 2.0))


def batch_sums(seq: np.ndarray, start: int, kappa: int, per_chain: int) -> np.ndarray:
    """Per-chain sums of per_chain consecutive kappa-batches from `start`
    (seq: [omega x length] 0/1 samples)."""
    out = np.zeros((seq.shape[0], per_chain), dtype=np.int64)
    for c in range(seq.shape[0]):
        a = np.asarray(seq[c, start:start + kappa * per_chain], dtype=np.int64)
        out[c] = a.reshape(per_chain, kappa).sum(axis=1)
    return out


def parallel_skart(model, pred, seed: int, omega: int, psi0: int, threshold: float, h_star: float,
                   alpha_conf: float, max_steps: int, threads: int = 8, source=None) -> RunResult:
    """Algorithm 5 with SPEC's declared Skart constants (reading
    Q11) and omega-rounded batch counts (Q12).  `trace` lists, per randomness
    test, (kappa, p, d, z, passed) and finally ("ci", kappa, p, d)."""
    ch = source if source is not None else Chains(model, pred, seed, omega, threads)
    psi, rhat, it, window = generate_converged_chains(ch, psi0, threshold, max_steps)
    seq = np.array(window, dtype=np.uint8)           # post-burn-in samples (skip first psi), [omega x length]

    def ensure(per_chain_len: int):
        nonlocal seq
        need = per_chain_len - seq.shape[1]
        if need > 0:
            if ch.length + need > max_steps:
                raise RuntimeError("Skart sample exceeds the step cap")
            I = ch.advance(0, need)
            seq = np.concatenate([seq, np.asarray(I, np.uint8)], axis=1)

    z_pass = ost.inv_norm_cdf(1.0 - RANDOMNESS_LEVEL / 2.0)
    eta = -(-1280 // omega) * omega                 # line 3
    ensure(eta // omega)
    allx = seq[:, :eta // omega].ravel()
    B = skewness(allx)                              # line 5, all samples
    kappa = 1 if (not math.isnan(B) and abs(B) <= SKEW_LIMIT) else 16
    p = -(-eta // omega) * omega                    # line 6
    eta = kappa * p
    d = 0
    trace = []
    # lines 7-12: randomness test on spaced batch means
    for _ in range(MAX_SKART_ITERS):
        ensure(eta // omega)
        per = p // omega
        bs = batch_sums(seq, 0, kappa, per) / kappa
        spaced = bs[:, ::d + 1]
        z = von_neumann_z(spaced)
        trace.append((kappa, p, d, z, abs(z) <= z_pass))
        if abs(z) <= z_pass:
            break
        kappa = int(math.ceil(math.sqrt(2.0) * kappa))
        d += 1
        p = -(-p // omega) * omega
        eta = kappa * p
    # lines 13-21: CI loop on non-spaced batch means
    for _ in range(MAX_SKART_ITERS):
        ensure(eta // omega)
        per = p // omega
        ci = osk.ci_from_batches(batch_sums(seq, 0, kappa, per), kappa, alpha_conf)
        if ci.H <= h_star:
            return RunResult(estimate=ci.mu, rhat=rhat, psi=psi, steps_per_chain=ch.length,
                             gr_iterations=it, sample_size=eta, ci_lo=ci.ci_lo, ci_hi=ci.ci_hi,
                             M=kappa, N=p, extensions=d, psi_gr=psi, trace=trace + [("ci", kappa, p, d)])
        g = (ci.H / h_star) ** 2
        new_eta = int(math.ceil(g * eta))
        if p < P_CEILING:
            p = min(P_CEILING, int(math.ceil(g * p)))
        p = -(-p // omega) * omega
        kappa = max(kappa, -(-new_eta // p))
        eta = kappa * p
    raise RuntimeError("Skart did not reach the precision within the iteration cap")
