"""Statistical pins: long oracle trajectories vs the exact steady state.

Catches mistakes anywhere in the oracle's simulator (stream, thresholds,
selection, lookup, commit, perturbation semantics, predicate) that the
exact matrix builders (written independently from the definitions) do not
share.  Tolerance: 4.5 batch-means standard errors (S:173 uses 3; a wider
band keeps the false-failure rate of the whole suite negligible).
"""
import numpy as np
import pytest

from oracle import exact, sim
from workloads import Predicate, config_model, config_predicate, random_pbn


def _check_freq(I: np.ndarray, target: float, nsig: float = 4.5):
    # I: chains x steps; batch means over 50 batches per chain
    chains, steps = I.shape
    nb = 50
    bm = I[:, : steps // nb * nb].reshape(chains, nb, -1).mean(axis=2).ravel()
    est = bm.mean()
    se = bm.std(ddof=1) / np.sqrt(len(bm))
    assert abs(est - target) < nsig * se + 1e-12, (est, target, se)


@pytest.mark.parametrize("per_node", [False, True])
def test_tiny_model_property_frequency(per_node):
    m = random_pbn(4, 1, 3, 1, 3, 0.08, seed=21)
    pred = Predicate(np.array([0, 3], np.uint16), np.array([1, 0], np.uint8))
    pi = exact.lu_solve(exact.matrix_product_form(m, per_node))
    target = exact.property_probability(pi, m.n, pred)
    _, I = sim.simulate(m, pred, seed=3, chain_ids=np.arange(4), step0=0, burn_in=200,
                        steps=100_000, per_node=per_node, threads=4)
    _check_freq(I, target)


def test_tiny_model_full_state_distribution():
    m = random_pbn(3, 2, 3, 0, 3, 0.1, seed=8)
    pi = exact.lu_solve(exact.matrix_product_form(m))
    # one predicate per state: all 8 indicator frequencies
    for s in range(8):
        pred = Predicate(np.arange(3, dtype=np.uint16),
                         np.array([(s >> i) & 1 for i in range(3)], np.uint8))
        _, I = sim.simulate(m, pred, seed=11 + s, chain_ids=np.arange(2), step0=0,
                            burn_in=100, steps=60_000, threads=2)
        _check_freq(I, pi[s])


def test_C1_property_frequency_vs_exact_1024_states():
    """BASELINE C1: exact steady state by power iteration on the 1024-state
    matrix; long oracle chains within 4.5 sigma."""
    m = config_model("C1")
    pred = config_predicate("C1")
    T = exact.matrix_product_form(m)
    pi = exact.power_iteration(T)
    target = exact.property_probability(pi, m.n, pred)
    _, I = sim.simulate(m, pred, seed=1, chain_ids=np.arange(8), step0=0, burn_in=1000,
                        steps=100_000, threads=8)
    _check_freq(I, target)


def test_perturbation_rate():
    """Fraction of VECTOR steps that are pure XOR perturbations equals
    1-(1-p)^n: use an all-constant-0 network, where a step leaves
    the all-zero state iff some gamma_i = 1."""
    from workloads import model_from_lists
    n, p = 6, 0.02
    m = model_from_lists(n, p, [[([], [0], 1.0)] for _ in range(n)])
    # predicate "state is all zero"; after any step from all-zero, I=0 iff perturbed.
    pred = Predicate(np.arange(n, dtype=np.uint16), np.zeros(n, np.uint8))
    # each step starts from all-zero only when the previous state was reset by
    # the functions; count I=0 among steps whose predecessor had I=1
    _, I = sim.simulate(m, pred, seed=2, chain_ids=np.arange(4), step0=0, burn_in=1,
                        steps=200_000, threads=4)
    prev, nxt = I[:, :-1], I[:, 1:]
    frm = prev == 1
    rate = float(np.sum(frm & (nxt == 0))) / float(np.sum(frm))
    pq, _ = exact.quantised_probs(m)
    target = 1 - (1 - pq) ** n
    k = float(np.sum(frm))
    assert abs(rate - target) < 4.5 * np.sqrt(target * (1 - target) / k)
