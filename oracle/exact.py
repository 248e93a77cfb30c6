"""Exact steady state of tiny PBNs -- TEST INFRASTRUCTURE ONLY.

The PBN with perturbations is an ergodic DTMC over S = {0,1}^n;
its steady state is lim pi_0 P^k.  Two independent builders of
the 2^n x 2^n transition matrix of the QUANTISED model (reading Q3: p and
c_j are the probabilities the 32-bit words realise):

  (a) product form: for VECTOR
        T(s,s') = [h>0] p^h (1-p)^(n-h) + (1-p)^n prod_i q_i(s)^{s'_i}(1-q_i(s))^{1-s'_i}
      with h = Hamming(s,s') and q_i(s) = sum_j c_j [f_j^(i)(s) = 1];
      for PER_NODE  T(s,s') = prod_i ( p [s'_i != s_i] + (1-p) P(f^(i)(s) = s'_i) );
  (b) brute-force enumeration of every realisation f_k and
      every perturbation vector gamma.

Stationary distribution by power iteration from any start and
by a dense LU solve of pi (P - I) = 0, sum pi = 1.

State encoding: integer s with bit i = value of node i.
"""
from __future__ import annotations

import itertools

import numpy as np


def quantised_probs(model):
    """(p_q, c_q) realised by the 32-bit word scheme (reading Q3).

    p_q = T_p / 2^32; given no perturbation the word is uniform on
    [T_p, 2^32) and function j is chosen on [D_{j-1}, D_j) with D_0 = T_p,
    D_ell = 2^32, so c_q[j] = (D_j - D_{j-1}) / (2^32 - T_p).
    Computed here from the definitions in exact integer arithmetic
    (independent of oracle/pbn_oracle.c's code).
    """
    two32 = 1 << 32
    Tp = int(np.floor(np.ldexp(model.p, 32)))
    span = two32 - Tp
    c_q = np.zeros(model.nf)
    for i in range(model.n):
        f0, f1 = int(model.fn_off[i]), int(model.fn_off[i + 1])
        prevD = Tp
        C = 0.0
        for f in range(f0, f1):
            C = C + float(model.sel_prob[f])
            if f == f1 - 1:
                D = two32
            else:
                Q = min(int(np.floor(np.ldexp(C, 32))), two32)
                D = Tp + (Q * span) // two32
            c_q[f] = (D - prevD) / span
            prevD = D
    return Tp / two32, c_q


def _fn_value(model, f: int, s: int) -> int:
    idx = 0
    for par in model.fn_parents(f):
        idx = idx * 2 + ((s >> par) & 1)
    return model.fn_table_bit(f, idx)


def matrix_product_form(model, per_node: bool = False) -> np.ndarray:
    n = model.n
    S = 1 << n
    p, c = quantised_probs(model)
    # q[s, i] = probability that node i's selected function outputs 1
    q = np.zeros((S, n))
    for s in range(S):
        for i in range(n):
            q[s, i] = sum(c[f] * _fn_value(model, f, s)
                          for f in range(model.fn_off[i], model.fn_off[i + 1]))
    states = np.arange(S)
    bits = ((states[:, None] >> np.arange(n)[None, :]) & 1).astype(np.float64)  # [s', i]
    T = np.zeros((S, S))
    for s in range(S):
        sb = bits[s]
        if per_node:
            fprob = bits * q[s][None, :] + (1 - bits) * (1 - q[s][None, :])  # P(f(s)_i = s'_i)
            flip = (bits != sb[None, :]).astype(np.float64)
            T[s] = np.prod(p * flip + (1 - p) * fprob, axis=1)
        else:
            h = np.sum(bits != sb[None, :], axis=1)
            pert = np.where(h > 0, p ** h * (1 - p) ** (n - h), 0.0)
            fn = np.prod(bits * q[s][None, :] + (1 - bits) * (1 - q[s][None, :]), axis=1)
            T[s] = pert + (1 - p) ** n * fn
    return T


def matrix_enumeration(model, per_node: bool = False) -> np.ndarray:
    """Brute force over realisations x perturbation vectors (tiny n only)."""
    n = model.n
    S = 1 << n
    p, c = quantised_probs(model)
    choices = [range(model.fn_off[i], model.fn_off[i + 1]) for i in range(n)]
    T = np.zeros((S, S))
    for s in range(S):
        for real in itertools.product(*choices):
            w_real = 1.0
            for f in real:
                w_real *= c[f]
            fs = [_fn_value(model, f, s) for f in real]
            for gamma in range(S):
                h = bin(gamma).count("1")
                w = w_real * p ** h * (1 - p) ** (n - h)
                if per_node:
                    nxt = 0
                    for i in range(n):
                        bit = (1 - ((s >> i) & 1)) if (gamma >> i) & 1 else fs[i]
                        nxt |= bit << i
                elif gamma != 0:
                    nxt = s ^ gamma
                else:
                    nxt = sum(fs[i] << i for i in range(n))
                T[s, nxt] += w
    return T


def power_iteration(T: np.ndarray, start: np.ndarray | None = None, tol: float = 1e-13,
                    max_iter: int = 10_000_000) -> np.ndarray:
    S = T.shape[0]
    pi = np.full(S, 1.0 / S) if start is None else np.asarray(start, dtype=np.float64)
    for _ in range(max_iter):
        nxt = pi @ T
        if np.max(np.abs(nxt - pi)) < tol:
            return nxt / nxt.sum()
        pi = nxt
    raise RuntimeError("power iteration did not converge")


def lu_solve(T: np.ndarray) -> np.ndarray:
    S = T.shape[0]
    A = T.T - np.eye(S)
    A[-1, :] = 1.0          # replace one balance equation by sum pi = 1
    b = np.zeros(S)
    b[-1] = 1.0
    return np.linalg.solve(A, b)


def property_probability(pi: np.ndarray, n: int, pred) -> float:
    tot = 0.0
    for s in range(1 << n):
        if all(((s >> int(node)) & 1) == int(v) for node, v in zip(pred.nodes, pred.values)):
            tot += pi[s]
    return tot


# --------------------------------------------------------------------------
# Geometric-skip perturbation stream (NEXT-2, reading Q18), VECTOR
# semantics: gamma(t) is drawn as the positions of its ones by successive
# geometric skips G(v) = #{g < n : Cg[g] <= v}, Cg[g] = floor((1 - q^(g+1))
# 2^32), q = 1 - p (q^(g+1) by repeated fp64 multiplication); with gamma = 0
# the nodes select with the unperturbed thresholds Q_j (T_p = 0).
# --------------------------------------------------------------------------
def geometric_cdf_table(model) -> list[int]:
    q, r, out = 1.0 - float(model.p), 1.0, []
    for _g in range(model.n):
        r = r * q
        out.append(int(np.floor(np.ldexp(1.0 - r, 32))))
    return out


def _skip_probs(model):
    """P(G = g) for g < n and P(G >= L) for L = 0..n, as exact fractions of 2^32."""
    C = geometric_cdf_table(model)
    two32 = 1 << 32
    eq = [(C[g] - (C[g - 1] if g else 0)) / two32 for g in range(model.n)]
    ge = [1.0] + [(two32 - C[L - 1]) / two32 for L in range(1, model.n + 1)]
    return eq, ge


def geometric_gamma_distribution(model) -> np.ndarray:
    """P(gamma = v) for every v in {0,1}^n (bit i = node i), closed form:
    the product of the skip probabilities of v's gaps and of the final
    skip past node n-1."""
    n = model.n
    eq, ge = _skip_probs(model)
    P = np.zeros(1 << n)
    for v in range(1 << n):
        ones = [i for i in range(n) if (v >> i) & 1]
        pr, prev = 1.0, -1
        for k in ones:
            pr *= eq[k - prev - 1]
            prev = k
        pr *= ge[n - prev - 1]
        P[v] = pr
    return P


def geometric_gamma_by_enumeration(model) -> np.ndarray:
    """The same distribution by enumerating every outcome of the skip
    process (draw after draw) -- an independent construction."""
    n = model.n
    eq, ge = _skip_probs(model)
    P = np.zeros(1 << n)

    def walk(k, v, pr):       # next candidate position k, flips so far v
        P_stop = ge[n - k]     # G >= n - k: no further flip
        P[v] += pr * P_stop
        for g in range(n - k):
            walk(k + g + 1, v | (1 << (k + g)), pr * eq[g])

    walk(0, 0, 1.0)
    return P


def unperturbed_selection_probs(model) -> np.ndarray:
    """c_q[f] realised by the node word with T_p = 0: (Q_j - Q_{j-1}) / 2^32."""
    two32 = 1 << 32
    c_q = np.zeros(model.nf)
    for i in range(model.n):
        f0, f1 = int(model.fn_off[i]), int(model.fn_off[i + 1])
        prevQ, C = 0, 0.0
        for f in range(f0, f1):
            C = C + float(model.sel_prob[f])
            Q = two32 if f == f1 - 1 else min(int(np.floor(np.ldexp(C, 32))), two32)
            c_q[f] = (Q - prevQ) / two32
            prevQ = Q
    return c_q


def matrix_geometric(model, gamma_probs=None) -> np.ndarray:
    """T(s, s') = P_gamma(s XOR s') [s' != s] + P_gamma(0) prod_i P(f_i(s) = s'_i)
    (VECTOR semantics, with gamma from the skip stream)."""
    n = model.n
    S = 1 << n
    Pg = geometric_gamma_distribution(model) if gamma_probs is None else gamma_probs
    c = unperturbed_selection_probs(model)
    states = np.arange(S)
    bits = ((states[:, None] >> np.arange(n)[None, :]) & 1).astype(np.float64)
    T = np.zeros((S, S))
    for s in range(S):
        q = np.array([sum(c[f] * _fn_value(model, f, s) for f in range(model.fn_off[i], model.fn_off[i + 1]))
                      for i in range(n)])
        fn = np.prod(bits * q[None, :] + (1 - bits) * (1 - q[None, :]), axis=1)
        pert = Pg[states ^ s].copy()
        pert[s] = 0.0
        T[s] = pert + Pg[0] * fn
    return T
