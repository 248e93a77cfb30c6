"""Pins for oracle/exact.py.

Two independently built transition matrices must agree; the stationary
distribution from power iteration and from LU must agree; three closed
forms derived by hand must be reproduced.
"""
import math

import numpy as np
import pytest

from oracle import exact
from workloads import model_from_lists, random_pbn


def const(v, prob):
    return ([], [v], prob)


@pytest.mark.parametrize("per_node", [False, True])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_builders_agree(per_node, seed):
    m = random_pbn(3, 1, 3, 0, 3, 0.2, seed=seed)
    A = exact.matrix_product_form(m, per_node)
    B = exact.matrix_enumeration(m, per_node)
    assert np.allclose(A, B, atol=1e-15, rtol=0)
    assert np.allclose(A.sum(axis=1), 1.0, atol=1e-13)


def test_builders_agree_n4():
    m = random_pbn(4, 1, 2, 1, 2, 0.05, seed=9)
    for per_node in (False, True):
        assert np.allclose(exact.matrix_product_form(m, per_node),
                           exact.matrix_enumeration(m, per_node), atol=1e-15, rtol=0)


def test_power_iteration_equals_lu_and_is_start_independent():
    m = random_pbn(6, 1, 3, 1, 4, 0.02, seed=4)
    T = exact.matrix_product_form(m)
    pi_u = exact.power_iteration(T)
    pi_lu = exact.lu_solve(T)
    start = np.zeros(T.shape[0])
    start[17] = 1.0
    pi_pt = exact.power_iteration(T, start)
    assert np.allclose(pi_u, pi_lu, atol=1e-11)
    assert np.allclose(pi_u, pi_pt, atol=1e-11)
    assert abs(pi_u.sum() - 1) < 1e-12
    assert np.max(np.abs(pi_u @ T - pi_u)) < 1e-12


@pytest.mark.parametrize("per_node", [False, True])
def test_closed_form_n1_constants(per_node):
    # n=1, const-1 with prob q, const-0 with prob 1-q:
    # pi_1 = (p + (1-p) q) / (2p + (1-p)), both semantics
    for p, q in [(0.5, 0.25), (0.01, 0.7), (0.2, 0.5)]:
        m = model_from_lists(1, p, [[const(1, q), const(0, 1 - q)]])
        pq, cq = exact.quantised_probs(m)
        pi = exact.lu_solve(exact.matrix_product_form(m, per_node))
        qq = cq[0]
        assert math.isclose(pi[1], (pq + (1 - pq) * qq) / (2 * pq + (1 - pq)), rel_tol=1e-12)


@pytest.mark.parametrize("per_node", [False, True])
def test_closed_form_identity_network_uniform(per_node):
    # identity network: every node copies itself -> pi uniform
    n = 3
    m = model_from_lists(n, 0.1, [[([i], [0, 1], 1.0)] for i in range(n)])
    pi = exact.lu_solve(exact.matrix_product_form(m, per_node))
    assert np.allclose(pi, 1.0 / 2 ** n, atol=1e-13)


def test_closed_form_two_constant_one_nodes_distinguishes_semantics():
    # n=2, both nodes constant 1.
    # VECTOR:   pi(11) = (2p^3 - 2p^2 + p + 1) / ((3p + 1)(p^2 + 1))
    # PER_NODE: pi(11) = 1 / (1 + p)^2
    for p in [0.5, 0.25, 0.01]:
        m = model_from_lists(2, p, [[const(1, 1.0)], [const(1, 1.0)]])
        pq, _ = exact.quantised_probs(m)
        pv = exact.lu_solve(exact.matrix_product_form(m, False))
        pp = exact.lu_solve(exact.matrix_product_form(m, True))
        assert math.isclose(pv[3], (2 * pq**3 - 2 * pq**2 + pq + 1) / ((3 * pq + 1) * (pq**2 + 1)),
                            rel_tol=1e-12)
        assert math.isclose(pp[3], 1.0 / (1 + pq) ** 2, rel_tol=1e-12)
