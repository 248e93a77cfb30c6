"""GPU: the library's host driver (pbn_run: Algorithm 3 then 4 or 5) vs the
oracle drivers (oracle/driver.py) on the same seeded inputs.

Integer decisions (psi, iterations, extensions, sample sizes, M, N, batch
size and count) must be identical; fp64 statistics agree within 1e-9
relative (BASELINE north_star).
"""
import math

import numpy as np
import pytest

from oracle import driver as odr
from workloads import CONFIGS, Predicate, config_model, config_predicate, random_pbn

pytestmark = pytest.mark.gpu
REL = 1e-9


@pytest.fixture(scope="module")
def pbn():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1508_07828_b200 as pbn
    return pbn


def close(a, b, rel=REL):
    return math.isclose(a, b, rel_tol=rel, abs_tol=1e-300)


def run_both_two_state(pbn, model, pred, omega, psi0, thr, r, s, eps, seed, max_steps=1 << 22):
    pm = pbn.pbn_load(model)
    st, res, err = pbn.pbn_run(pm, method=0, omega=omega, psi0=psi0, rhat_threshold=thr, r=r, s=s, eps=eps,
                               seed=seed, pred=pred, max_steps=max_steps)
    assert st == 0, err
    o = odr.parallel_two_state(model, pred, seed, omega, psi0, thr, r, s, eps, max_steps, threads=16)
    return res, o


def check_two_state(res, o):
    assert (res.psi, res.gr_iterations, res.extensions, res.sample_size, res.steps_per_chain) == (
        o.psi, o.gr_iterations, o.extensions, o.sample_size, o.steps_per_chain)
    assert (res.M, res.N) == (o.M, o.N)
    assert close(res.rhat, o.rhat) and close(res.alpha, o.alpha) and close(res.beta, o.beta)
    assert close(res.estimate, o.estimate, 1e-12)


def test_two_state_driver_C1_model(pbn):
    model, pred = config_model("C1"), config_predicate("C1")
    res, o = run_both_two_state(pbn, model, pred, omega=8, psi0=500, thr=1.1, r=0.01, s=0.95, eps=1e-10,
                                seed=1)
    check_two_state(res, o)


def test_two_state_driver_burn_in_recheck(pbn):
    """A slowly mixing model with a tiny psi0 so that M > psi forces the
    Algorithm 4 burn-in re-check (discard + recount)."""
    nodes = [[([0], [0, 1], 1.0)], [([0, 1], [0, 1, 1, 1], 0.9), ([], [0], 0.1)]]
    from workloads import model_from_lists
    model = model_from_lists(2, 0.002, nodes)
    pred = Predicate(np.array([1], np.uint16), np.array([1], np.uint8))
    res, o = run_both_two_state(pbn, model, pred, omega=4, psi0=8, thr=1.5, r=0.02, s=0.95, eps=1e-10, seed=7)
    check_two_state(res, o)


def test_two_state_driver_burn_in_discard_past_the_sample(pbn):
    """a burn-in re-check whose M - psi exceeds the current sample
    (identity network, alpha = beta = p = 1e-3, omega = 16, r = 0.1): the
    discard continues into the next extension, in the library
    driver exactly as in the oracle's (pinned by re-simulation in
    test_oracle_driver_pins.py)."""
    from workloads import model_from_lists
    model = model_from_lists(1, 0.001, [[([0], [0, 1], 1.0)]])
    pred = Predicate(np.array([0], np.uint16), np.array([1], np.uint8))
    res, o = run_both_two_state(pbn, model, pred, omega=16, psi0=8, thr=1.1, r=0.1, s=0.95, eps=1e-10, seed=3,
                                max_steps=1 << 24)
    assert any(t[3] > t[4] for t in o.trace)
    check_two_state(res, o)


def test_two_state_driver_C2_config(pbn):
    """BASELINE C2: 1024 chains, psi0 = 1000, R-hat < 1.1, r = 0.01, s = 0.95."""
    c = CONFIGS["C2"]
    x = c.extra
    res, o = run_both_two_state(pbn, config_model("C2"), config_predicate("C2"), omega=c.chains,
                                psi0=x["psi0"], thr=x["rhat_threshold"], r=x["r"], s=x["s"], eps=x["eps"],
                                seed=c.sim_seed)
    check_two_state(res, o)


@pytest.mark.parametrize("omega,seed", [(8, 3), (3, 5), (64, 2)])
def test_skart_driver(pbn, omega, seed):
    model = random_pbn(12, 1, 3, 1, 3, 0.02, seed=seed)
    pred = Predicate(np.array([0, 5], np.uint16), np.array([1, 0], np.uint8))
    pm = pbn.pbn_load(model)
    st, res, err = pbn.pbn_run(pm, method=1, omega=omega, psi0=256, rhat_threshold=1.1, h_star=0.01,
                               alpha_conf=0.05, seed=seed, pred=pred, max_steps=1 << 22)
    assert st == 0, err
    o = odr.parallel_skart(model, pred, seed, omega, 256, 1.1, 0.01, 0.05, 1 << 22, threads=16)
    assert (res.psi, res.gr_iterations, res.sample_size, res.steps_per_chain) == (
        o.psi, o.gr_iterations, o.sample_size, o.steps_per_chain)
    assert (res.M, res.N, res.extensions) == (o.M, o.N, o.extensions)     # kappa, p, spacer d
    for a, b in [(res.estimate, o.estimate), (res.ci_lo, o.ci_lo), (res.ci_hi, o.ci_hi), (res.rhat, o.rhat)]:
        assert close(a, b), (a, b)
    assert res.ci_lo <= res.estimate <= res.ci_hi


def _multi_props(model, q, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(q):
        k = int(rng.integers(1, 3))
        nodes = rng.choice(model.n, size=k, replace=False).astype(np.uint16)
        out.append(Predicate(nodes, rng.integers(0, 2, size=k).astype(np.uint8)))
    return out


@pytest.mark.parametrize("key,q,omega,psi0,seed", [("C1", 4, 8, 400, 1), ("C2", 7, 16, 500, 2)])
def test_multi_property_driver_matches_oracle(pbn, key, q, omega, psi0, seed):
    """pbn_run_multi (reading Q13) vs the oracle's multi-property
    Algorithm 4: identical integer decisions, per-property statistics within
    1e-9, and each estimate equals the pooled mean of its own meta states."""
    model = config_model(key)
    props = _multi_props(model, q, seed)
    pm = pbn.pbn_load(model)
    st, res, per, err = pbn.pbn_run_multi(pm, props, omega=omega, psi0=psi0, rhat_threshold=1.1, r=0.02,
                                          s=0.95, eps=1e-10, seed=seed, max_steps=1 << 22)
    assert st == 0, err
    o = odr.parallel_two_state_multi(model, props, seed, omega, psi0, 1.1, 0.02, 0.95, 1e-10, 1 << 22,
                                     threads=16)
    assert (res.psi, res.gr_iterations, res.extensions, res.sample_size, res.steps_per_chain) == (
        o.psi, o.gr_iterations, o.extensions, o.sample_size, o.steps_per_chain)
    assert close(res.rhat, o.rhat)
    for g, r in zip(per, o.per_prop):
        assert (g.status != 0) == r["degenerate"]
        assert close(g.estimate, r["estimate"], 1e-12)
        if not r["degenerate"]:
            assert (g.M, g.N) == (r["M"], r["N"])
            assert close(g.alpha, r["alpha"]) and close(g.beta, r["beta"])
    # every property's N is met by the pooled sample
    assert all(g.N <= res.sample_size for g, r in zip(per, o.per_prop) if not r["degenerate"])


def _sharded_rank(rank, world, port, outdir):
    import os
    import torch
    import torch.distributed as dist
    import paper_1508_07828_b200 as pbn
    from workloads import config_model, config_predicate
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    pm = pbn.pbn_load(config_model("C2"))
    st, res, err = pbn.parallel.run_sharded(pm, omega=24, psi0=500, rhat_threshold=1.1, r=0.02, s=0.95,
                                            eps=1e-10, seed=7, pred=config_predicate("C2"))
    np.save(os.path.join(outdir, f"r{rank}.npy"),
            np.array([st, res.psi, res.gr_iterations, res.extensions, res.sample_size, res.steps_per_chain,
                      res.M, res.N, res.estimate, res.rhat, res.alpha, res.beta], dtype=np.float64))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_driver_equals_single_gpu_run(pbn):
    """pbn_run_sharded (chains split over 2 ranks, 6-u64 all-reduce per
    decision over gloo; both ranks on this GPU -- a functional check of the
    multi-GPU driver, not a performance run) gives every decision and
    statistic of the single-GPU pbn_run over all chains."""
    import socket
    import tempfile
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_sharded_rank, args=(2, port, d), nprocs=2, join=True)
        got = [np.load(f"{d}/r{r}.npy") for r in range(2)]
    pm = pbn.pbn_load(config_model("C2"))
    st, res, err = pbn.pbn_run(pm, method=0, omega=24, psi0=500, rhat_threshold=1.1, r=0.02, s=0.95,
                               eps=1e-10, seed=7, pred=config_predicate("C2"))
    assert st == 0, err
    ref = np.array([st, res.psi, res.gr_iterations, res.extensions, res.sample_size, res.steps_per_chain,
                    res.M, res.N, res.estimate, res.rhat, res.alpha, res.beta], dtype=np.float64)
    for g in got:
        assert np.array_equal(g, ref), (g, ref)


def test_skart_driver_C3_protocol(pbn):
    """BASELINE C3 (n = 1000, 4096 chains, Gelman-Rubin from psi0 = 5e4, i.e.
    10^5 transitions per chain, then Skart, H* = 1e-3, alpha = 0.05) end to
    end through pbn_run(SKART), against the oracle's Algorithm 3 + 5 decision
    code (oracle/driver.py) run on the same GPU trajectories (tests.helpers
    .GpuChains; the trajectories are bit-exact to the oracle simulator on 64
    sampled chains in test_parity_gpu.py): identical psi, kappa, p, spacer
    and steps, estimate / CI / R-hat within 1e-9."""
    from tests.helpers import GpuChains
    c = CONFIGS["C3"]
    model, pred = config_model("C3"), config_predicate("C3")
    pm = pbn.pbn_load(model)
    kw = dict(omega=c.chains, psi0=c.burn_in, rhat_threshold=1.1, h_star=1e-3, alpha_conf=0.05, seed=c.sim_seed,
              pred=pred, max_steps=1 << 22)
    st, res, err = pbn.pbn_run(pm, method=1, **kw)
    assert st == 0, err
    src = GpuChains(pbn, pm, pred, c.sim_seed, c.chains)
    o = odr.parallel_skart(model, pred, c.sim_seed, c.chains, c.burn_in, 1.1, 1e-3, 0.05, 1 << 22, source=src)
    assert (res.psi, res.gr_iterations, res.sample_size, res.steps_per_chain) == (
        o.psi, o.gr_iterations, o.sample_size, o.steps_per_chain)
    assert (res.M, res.N, res.extensions) == (o.M, o.N, o.extensions)
    for a, b in [(res.estimate, o.estimate), (res.ci_lo, o.ci_lo), (res.ci_hi, o.ci_hi), (res.rhat, o.rhat)]:
        assert close(a, b), (a, b)


@pytest.mark.parametrize("omega,seed", [(8, 3), (5, 11)])
def test_pbn_skart_boundary_call(pbn, omega, seed):
    """pbn_skart (C ABI) over device bitstreams, called with a growing
    sample until it stops asking for more, against the oracle's Algorithm 5
    decisions on the same trajectories."""
    import torch
    from tests.helpers import GpuChains
    model = random_pbn(12, 1, 3, 1, 3, 0.02, seed=seed)
    pred = Predicate(np.array([0, 5], np.uint16), np.array([1, 0], np.uint8))
    pm = pbn.pbn_load(model)
    o = odr.parallel_skart(model, pred, seed, omega, 256, 1.1, 0.01, 0.05, 1 << 22,
                           source=GpuChains(pbn, pm, pred, seed, omega))
    psi = o.psi
    # the chains after Algorithm 3: 2 psi transitions, sample = the last psi
    avail, calls = psi, 0
    while True:
        total = psi + avail
        out = pbn.alloc_outputs(pm, omega, total, emit_bits=True)
        pbn.pbn_simulate(pm, out, n_chains=omega, steps=total, seed=seed, pred=pred, init=True, emit_bits=True)
        torch.cuda.synchronize()
        st, r = pbn.pbn_skart(out.bits, omega, out.bits.shape[1], psi, avail, 0.01, 0.05)
        calls += 1
        if st == 0:
            break
        assert st == 4 and r.need_per_chain > avail, (st, r.need_per_chain)
        avail = r.need_per_chain
    assert psi + avail == o.steps_per_chain
    assert (r.kappa, r.batches, r.spacer, r.eta) == (o.M, o.N, o.extensions, o.sample_size)
    for a, b in [(r.estimate, o.estimate), (r.ci_lo, o.ci_lo), (r.ci_hi, o.ci_hi)]:
        assert close(a, b), (a, b)


def _sharded_skart_rank(rank, world, port, outdir):
    import os
    import torch
    import torch.distributed as dist
    import paper_1508_07828_b200 as pbn
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    model = random_pbn(12, 1, 3, 1, 3, 0.02, seed=3)
    pred = Predicate(np.array([0, 5], np.uint16), np.array([1, 0], np.uint8))
    pm = pbn.pbn_load(model)
    st, res, err = pbn.parallel.run_sharded(pm, omega=9, psi0=256, rhat_threshold=1.1, seed=3, pred=pred,
                                            method=1, h_star=0.01, alpha_conf=0.05, max_steps=1 << 22)
    np.save(os.path.join(outdir, f"r{rank}.npy"),
            np.array([st, res.psi, res.gr_iterations, res.extensions, res.sample_size, res.steps_per_chain,
                      res.M, res.N, res.estimate, res.rhat, res.ci_lo, res.ci_hi], dtype=np.float64))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_skart_equals_single_gpu_run(pbn):
    """Skart over chains sharded on 2 ranks (9 chains: 5 + 4; per-chain batch
    sums all-gathered, Fig. 2b) gives the single-GPU pbn_run's decisions and
    CI bit for bit."""
    import socket
    import tempfile
    import torch.multiprocessing as mp
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_sharded_skart_rank, args=(2, port, d), nprocs=2, join=True)
        got = [np.load(f"{d}/r{r}.npy") for r in range(2)]
    model = random_pbn(12, 1, 3, 1, 3, 0.02, seed=3)
    pred = Predicate(np.array([0, 5], np.uint16), np.array([1, 0], np.uint8))
    pm = pbn.pbn_load(model)
    st, res, err = pbn.pbn_run(pm, method=1, omega=9, psi0=256, rhat_threshold=1.1, h_star=0.01, alpha_conf=0.05,
                               seed=3, pred=pred, max_steps=1 << 22)
    assert st == 0, err
    ref = np.array([st, res.psi, res.gr_iterations, res.extensions, res.sample_size, res.steps_per_chain,
                    res.M, res.N, res.estimate, res.rhat, res.ci_lo, res.ci_hi], dtype=np.float64)
    for g in got:
        assert np.array_equal(g, ref), (g, ref)
