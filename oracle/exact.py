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
