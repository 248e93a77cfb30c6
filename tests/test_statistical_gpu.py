"""GPU statistical pins at scale (SURVEY §8(c)(iii) "MC vs exact"): >= 10^9
chain-steps of the CUDA path on tiny networks against the exact steady state
of the 2^n transition matrix (oracle/exact.py, power iteration / LU).

Bit-exactness against the oracle is checked elsewhere on small and sampled
runs; these tests exercise the full launch shapes (many groups, persistent
chunks, multi-property warps) over a billion steps and compare what the
paper's method estimates -- the steady-state probability of a property --
with its exact value, within 4.5 batch-means standard errors.
"""
import numpy as np
import pytest

from oracle import exact
from workloads import Predicate, config_model, config_predicate, random_pbn

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pbn():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1508_07828_b200 as pbn
    return pbn


def _batch_means_check(batch_sums: np.ndarray, kappa: int, target: float, nsig: float = 4.5):
    bm = batch_sums.astype(np.float64).ravel() / kappa
    est = bm.mean()
    se = bm.std(ddof=1) / np.sqrt(bm.size)
    assert abs(est - target) < nsig * se + 1e-12, (est, target, se)
    return est, se


def _run(pbn, model, props, chains, steps, burn_in, kappa, seed, per_node=False):
    import torch
    pm = pbn.pbn_load(model, per_node=per_node)
    out = pbn.alloc_outputs(pm, chains, steps, batch=kappa, n_props=len(props))
    pbn.pbn_simulate(pm, out, n_chains=chains, steps=steps, burn_in=burn_in, batch=kappa, seed=seed,
                     init=True, props=props)
    torch.cuda.synchronize()
    bs = out.batch_sums.cpu().numpy().view(np.uint32)
    pm.close()
    return bs


@pytest.mark.parametrize("per_node", [False, True])
def test_C1_billion_steps_vs_exact_steady_state(pbn, per_node):
    """BASELINE C1 network: 8192 chains x 125 000 steps (1.0e9 chain-steps);
    the property frequency against pi from the 1024-state matrix."""
    m, pred = config_model("C1"), config_predicate("C1")
    pi = exact.power_iteration(exact.matrix_product_form(m, per_node))
    target = exact.property_probability(pi, m.n, pred)
    bs = _run(pbn, m, [pred], chains=8192, steps=125_000, burn_in=2000, kappa=2500, seed=31, per_node=per_node)
    _batch_means_check(bs[0], 2500, target)


def test_every_state_frequency_in_one_launch(pbn):
    """A 3-node network, one property per state (8 properties evaluated by
    8 statistics warps on the same trajectories): all 8 state frequencies
    against the exact stationary distribution."""
    m = random_pbn(3, 2, 3, 0, 3, 0.1, seed=8)
    pi = exact.lu_solve(exact.matrix_product_form(m))
    props = [Predicate(np.arange(3, dtype=np.uint16), np.array([(s >> i) & 1 for i in range(3)], np.uint8))
             for s in range(8)]
    bs = _run(pbn, m, props, chains=4096, steps=250_000, burn_in=500, kappa=5000, seed=32)
    est = [_batch_means_check(bs[s], 5000, pi[s])[0] for s in range(8)]
    assert abs(sum(est) - 1.0) < 1e-12  # every state is in exactly one property
