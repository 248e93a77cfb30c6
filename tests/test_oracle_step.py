"""Pins for the oracle's thresholds and single step (PAPER §2.2).

Pinned by: SPEC worked examples, exact rational
arithmetic for the quantised thresholds (reading Q3), and empirical
one-step transition frequencies against the independently built exact
transition matrix (oracle/exact.py builders).
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle import exact, sim
from workloads import model_from_lists, random_pbn

TWO32 = 1 << 32


def const_fn(v):
    return ([], [v], 1.0)


def test_perturbation_threshold_exact():
    for p in [0.5, 2.0 ** -32, 0.01, 1e-4, 5e-5, 0.001, 0.3, 1 - 2.0 ** -20]:
        expect = int(Fraction(p) * TWO32)  # floor of the exact rational
        assert sim.perturbation_threshold(p) == expect


def test_selection_thresholds_closed_forms():
    # ell = 1: single function, no threshold but the terminal 2^32
    m = model_from_lists(2, 0.01, [[([0], [0, 1], 1.0)], [([1], [1, 0], 1.0)]])
    assert list(sim.selection_thresholds(m)) == [TWO32, TWO32]
    # c = (1/2, 1/2): D_1 = T_p + floor(2^31 (2^32 - T_p) / 2^32)
    p = 0.01
    m = model_from_lists(1, p, [[const_fn(0)[:2] + (0.5,), const_fn(1)[:2] + (0.5,)]])
    Tp = int(Fraction(p) * TWO32)
    D = sim.selection_thresholds(m)
    assert int(D[0]) == Tp + (2**31 * (TWO32 - Tp)) // TWO32
    assert int(D[1]) == TWO32


def test_thresholds_random_models_invariants():
    m = random_pbn(200, 1, 6, 1, 3, 1e-3, seed=11)
    D = sim.selection_thresholds(m)
    Tp = sim.perturbation_threshold(m.p)
    p_q, c_q = exact.quantised_probs(m)
    assert p_q == Tp / TWO32
    for i in range(m.n):
        f0, f1 = m.fn_off[i], m.fn_off[i + 1]
        d = [int(x) for x in D[f0:f1]]
        assert d[-1] == TWO32
        assert all(Tp <= x for x in d)
        assert all(a < b for a, b in zip(d[:-1], d[1:]))     # strictly increasing
        # quantised selection probabilities within 2^-31 of the model's
        assert np.allclose(c_q[f0:f1], m.sel_prob[f0:f1], atol=2.0 ** -31, rtol=0)
        # and they sum to one
        assert abs(c_q[f0:f1].sum() - 1.0) < 1e-12


def test_spec_s148_constant_true_forced_no_perturbation():
    n = 5
    m = model_from_lists(n, 0.01, [[const_fn(1)] for _ in range(n)])
    u = np.full(n, 0xFFFFFFFF, np.uint32)          # every word >= T_p: gamma = 0
    for s in [np.zeros(n, np.uint8), np.array([1, 0, 1, 0, 1], np.uint8)]:
        assert list(sim.step(m, s, u)) == [1] * n
        assert list(sim.step(m, s, u, per_node=True)) == [1] * n


def test_spec_s149_forced_gamma_xor():
    # forced gamma = (0,1,0) on s = (1,0,1) -> (1,1,1) under VECTOR
    n = 3
    m = model_from_lists(n, 0.01, [[const_fn(0)] for _ in range(n)])
    s = np.array([1, 0, 1], np.uint8)
    u = np.array([0xFFFFFFFF, 0, 0xFFFFFFFF], np.uint32)
    assert list(sim.step(m, s, u)) == [1, 1, 1]
    # PER_NODE (reading Q1): node 1 flips, nodes 0 and 2 apply const-0
    assert list(sim.step(m, s, u, per_node=True)) == [0, 1, 0]


def test_table_index_msb_is_first_parent():
    # f(x_a, x_b) with parents [2, 0]: idx = 2*s[2] + s[0]; table '0010' -> only idx 1 is true
    m = model_from_lists(3, 1e-3, [[([2, 0], [0, 1, 0, 0], 1.0)], [const_fn(0)], [const_fn(0)]])
    u = np.full(3, 0xFFFFFFFF, np.uint32)
    # s0=1, s2=0 -> idx = 0b01 = 1 -> 1
    assert sim.step(m, np.array([1, 0, 0], np.uint8), u)[0] == 1
    # s0=0, s2=1 -> idx = 0b10 = 2 -> 0
    assert sim.step(m, np.array([0, 0, 1], np.uint8), u)[0] == 0


def test_selection_boundaries_given_thresholds():
    m = model_from_lists(1, 0.01, [[const_fn(0)[:2] + (0.3,), const_fn(1)[:2] + (0.7,)]])
    Tp = sim.perturbation_threshold(m.p)
    D1 = int(sim.selection_thresholds(m)[0])
    s = np.zeros(1, np.uint8)
    assert sim.step(m, s, np.array([Tp - 1], np.uint32))[0] == 1      # perturbed: 0 xor 1
    assert sim.step(m, s, np.array([Tp], np.uint32))[0] == 0          # function 1 (const 0)
    assert sim.step(m, s, np.array([D1 - 1], np.uint32))[0] == 0
    assert sim.step(m, s, np.array([D1], np.uint32))[0] == 1          # function 2 (const 1)


@pytest.mark.parametrize("per_node", [False, True])
def test_one_step_rows_match_exact_matrix(per_node):
    """Empirical one-step rows of the oracle step with Philox words vs the
    product-form matrix row, chi-square over all 2^n targets."""
    m = random_pbn(3, 1, 3, 0, 3, 0.15, seed=5)
    T = exact.matrix_product_form(m, per_node=per_node)
    n = m.n
    draws = 40_000
    for s_int in [0, 5]:
        s = np.array([(s_int >> i) & 1 for i in range(n)], np.uint8)
        counts = np.zeros(1 << n)
        for t in range(1, draws + 1):
            u = np.array([sim.word(99, s_int, t, i) for i in range(n)], np.uint32)
            nxt = sim.step(m, s, u, per_node=per_node)
            counts[int(sum(int(b) << i for i, b in enumerate(nxt)))] += 1
        exp = T[s_int] * draws
        mask = exp > 5
        chi2 = float(np.sum((counts[mask] - exp[mask]) ** 2 / exp[mask]))
        dof = int(mask.sum()) - 1
        assert chi2 < dof + 6 * np.sqrt(2 * dof) + 10, (chi2, dof)
        assert counts[~mask].sum() <= max(10, 3 * exp[~mask].sum() + 10)
