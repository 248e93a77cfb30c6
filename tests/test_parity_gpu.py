"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact
on every output field (state, c1, n01, n10, first/last, batch sums, bits,
totals) -- BASELINE north_star: "GPU trajectories, counts and transition
tallies must be bit-exact against the oracle".

Small configs are compared on all chains; C3-C5 run in the exact launch
configuration bench.py times and are compared on a deterministic sample of
chains that the oracle computes one by one at the full step count.
"""
import os

import numpy as np
import pytest

from tests.helpers import compare_chain, gpu_run, oracle_run, pack_states, sample_chain_ids, unpack_states
from oracle import stats as ostats
from workloads import (CONFIGS, Predicate, config_model, config_predicate, model_from_lists,
                       random_pbn)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pbn():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1508_07828_b200 as pbn
    return pbn


def load(pbn, model, per_node=False):
    return pbn.pbn_load(model, per_node=per_node)


def full_compare(pbn, model, pred, *, n_chains, steps, burn_in=0, seed=1, batch=0, per_node=False,
                 groups=0, warps=0, threads=8, cluster_size=0):
    pm = load(pbn, model, per_node)
    g = gpu_run(pm, model, pred, n_chains=n_chains, steps=steps, burn_in=burn_in, seed=seed,
                batch=batch, groups=groups, warps=warps, cluster_size=cluster_size)
    st, I, ws = oracle_run(model, pred, np.arange(n_chains), steps=steps, burn_in=burn_in, seed=seed,
                           batch=batch, per_node=per_node, threads=threads)
    packed = pack_states(st)
    for c in range(n_chains):
        compare_chain(g, c, packed[c], ws[c], steps, batch)
    assert np.array_equal(g["totals"], ostats.totals(ws))
    return g


def test_C1_all_fields_bit_exact(pbn):
    c = CONFIGS["C1"]
    full_compare(pbn, config_model("C1"), config_predicate("C1"), n_chains=c.chains, steps=c.steps,
                 burn_in=c.burn_in, seed=c.sim_seed, batch=c.batch)


def test_C1_per_node_semantics(pbn):
    c = CONFIGS["C1"]
    full_compare(pbn, config_model("C1"), config_predicate("C1"), n_chains=c.chains, steps=c.steps,
                 burn_in=c.burn_in, seed=c.sim_seed, batch=c.batch, per_node=True)


def test_C2_all_chains(pbn):
    c = CONFIGS["C2"]
    full_compare(pbn, config_model("C2"), config_predicate("C2"), n_chains=c.chains, steps=c.steps,
                 burn_in=c.burn_in, seed=c.sim_seed, batch=c.batch)


@pytest.mark.parametrize("key,n_chains", [("C3", 0), ("C4", 0), ("C5", 1), ("C5", 64), ("C5", 1024), ("C5", 16384),
                                          ("C5", 65536)])
def test_large_configs_sampled_chains(pbn, key, n_chains):
    """Full launch in the configuration bench.py times (C3, C4; C5 at every
    chain count of its sweep, with the kernel pbn_simulate auto-selects
    there: clusters of 16 / 8 CTAs for 1-1024 chains, the global-image K1
    beyond); the oracle recomputes up to 64 sampled chains at the full step
    count; invariants on every chain."""
    c = CONFIGS[key]
    model, pred = config_model(key), config_predicate(key)
    n_chains = n_chains or c.chains
    steps, burn_in = c.steps, c.burn_in
    pm = load(pbn, model)
    # C3 / C4: the chain-lanes kernel K1 (layout 1); auto runs the bit-sliced
    # K1b there, compared at these shapes in tests/test_bitslice_gpu.py
    layout = 1 if key in ("C3", "C4") else 0
    g = gpu_run(pm, model, pred, n_chains=n_chains, steps=steps, burn_in=burn_in, seed=c.sim_seed,
                batch=c.batch, layout=layout)
    if layout == 1:
        assert pbn.pbn_last_kernel() == "K1"
    ids = sample_chain_ids(n_chains, k=64, seed=c.sim_seed)
    st, I, ws = oracle_run(model, pred, ids, steps=steps, burn_in=burn_in, seed=c.sim_seed,
                           batch=c.batch, threads=os.cpu_count() or 8)
    packed = pack_states(st)
    for k, cid in enumerate(ids):
        compare_chain(g, cid, packed[k], ws[k], steps, c.batch)
    # properties that must hold for every chain at any size
    c1 = g["c1"].astype(np.int64)
    fl = g["first_last"].astype(np.int64)
    first, last = fl & 1, fl >> 1
    assert np.array_equal(g["n01"].astype(np.int64) - g["n10"].astype(np.int64), last - first)
    assert np.array_equal(g["batch_sums"].astype(np.int64).sum(axis=1), c1)
    pop = np.unpackbits(g["bits"].view(np.uint8), axis=1).sum(axis=1)
    assert np.array_equal(pop, c1)
    tot = g["totals"].astype(object)
    assert tot[0] == int(c1.sum()) and tot[1] == int((c1.astype(object) ** 2).sum())
    assert tot[2] == int(g["n01"].astype(np.int64).sum()) and tot[3] == int(g["n10"].astype(np.int64).sum())
    assert tot[5] == int((c1 - last).sum()) and tot[4] == int(((steps - c1) - (1 - last)).sum())


ALL = ["state", "c1", "n01", "n10", "first_last", "batch_sums", "bits", "totals"]


@pytest.mark.parametrize("per_node", [False, True])
def test_launch_shape_independence(pbn, per_node):
    """cluster_size=1 forces the single-CTA kernel K1 (200 chains = 7 groups
    would otherwise auto-select the cluster kernel): K1's warp splits and
    its persistent chunking are compared with K1 one-CTA-per-group, and the
    auto (cluster) launch with both; the oracle checks the reference."""
    model, pred = config_model("C2"), config_predicate("C2")
    pm = load(pbn, model, per_node)
    kw = dict(n_chains=200, steps=700, burn_in=300, seed=9, batch=64)
    ref = gpu_run(pm, model, pred, cluster_size=1, schedule=1, **kw)
    auto = gpu_run(pm, model, pred, **kw)
    for k in ALL:
        assert np.array_equal(auto[k], ref[k]), ("auto", k)
    for warps in [1, 2, 5, 7, 8, 13, 25]:
        g = gpu_run(pm, model, pred, warps=warps, cluster_size=1, schedule=1, **kw)
        for k in ALL:
            assert np.array_equal(g[k], ref[k]), (warps, k)
    # persistent schedule: chunks straddle the burn-in end, batch and bit-word boundaries
    for chunk, warps in [(1, 4), (7, 25), (33, 3), (299, 0), (1000, 8), (0, 0)]:
        g = gpu_run(pm, model, pred, warps=warps, schedule=2, chunk_steps=chunk, cluster_size=1, **kw)
        for k in ALL:
            assert np.array_equal(g[k], ref[k]), ("persistent", chunk, warps, k)
    ids = sample_chain_ids(200, k=6, seed=9)
    st, I, ws = oracle_run(model, pred, ids, steps=700, burn_in=300, seed=9, batch=64, per_node=per_node)
    packed = pack_states(st)
    for j, cid in enumerate(ids):
        compare_chain(ref, cid, packed[j], ws[j], 700, 64)


@pytest.mark.parametrize("per_node", [False, True])
def test_persistent_ragged_group_leaves_no_gamma_bits(pbn, per_node):
    """a ragged last group (20007 chains: 7 real lanes in group
    625) whose chain-less lanes draw perturbations must not leak gamma bits
    into the next work unit of the same CTA (persistent schedule, short
    chunks so every CTA runs many units)."""
    model, pred = config_model("C2"), config_predicate("C2")
    pm = load(pbn, model, per_node)
    kw = dict(n_chains=20007, steps=300, burn_in=60, seed=4, batch=50, cluster_size=1)
    a = gpu_run(pm, model, pred, schedule=1, **kw)
    b = gpu_run(pm, model, pred, schedule=2, chunk_steps=13, **kw)
    for k in ALL:
        assert np.array_equal(a[k], b[k]), k
    ids = [0, 19999, 20000, 20006] + sample_chain_ids(20007, k=4, seed=2)
    st, I, ws = oracle_run(model, pred, ids, steps=300, burn_in=60, seed=4, batch=50, per_node=per_node)
    packed = pack_states(st)
    for j, cid in enumerate(ids):
        compare_chain(b, cid, packed[j], ws[j], 300, 50)


def test_persistent_schedule_large_group_count(pbn):
    """More groups than resident CTAs (the C4 situation) with VECTOR and PER_NODE."""
    model, pred = config_model("C2"), config_predicate("C2")
    for per_node in (False, True):
        pm = load(pbn, model, per_node)
        a = gpu_run(pm, model, pred, n_chains=20000, steps=150, burn_in=50, seed=3, batch=16, schedule=1)
        b = gpu_run(pm, model, pred, n_chains=20000, steps=150, burn_in=50, seed=3, batch=16, schedule=2,
                    chunk_steps=37)
        for k in ["state", "c1", "n01", "n10", "first_last", "batch_sums", "bits", "totals"]:
            assert np.array_equal(a[k], b[k]), (per_node, k)
        ids = sample_chain_ids(20000, k=6, seed=1)
        st, I, ws = oracle_run(model, pred, ids, steps=150, burn_in=50, seed=3, batch=16, per_node=per_node)
        packed = pack_states(st)
        for j, cid in enumerate(ids):
            compare_chain(b, cid, packed[j], ws[j], 150, 16)


@pytest.mark.parametrize("cluster_size", [1, 0])
def test_chain_split_and_step_split(pbn, cluster_size):
    model, pred = config_model("C2"), config_predicate("C2")
    pm = load(pbn, model)
    cs = dict(cluster_size=cluster_size)
    full = gpu_run(pm, model, pred, n_chains=100, steps=640, burn_in=0, seed=5, batch=0, **cs)
    # chains 0..36 and 37..99 in separate calls (chain_base)
    a = gpu_run(pm, model, pred, n_chains=37, steps=640, seed=5, **cs)
    b = gpu_run(pm, model, pred, n_chains=63, chain_base=37, steps=640, seed=5, **cs)
    for k in ["state", "c1", "n01", "n10", "first_last", "bits"]:
        assert np.array_equal(np.concatenate([a[k], b[k]]), full[k]), k
    # steps 0..300 then 301..640 continuing the state; bits appended at an offset
    s1 = gpu_run(pm, model, pred, n_chains=100, steps=300, seed=5, bits_row_words=20, **cs)
    s2 = gpu_run(pm, model, pred, n_chains=100, steps=340, step0=300, seed=5, init=False,
                 state=s1["state"], bits_offset=300, bits_row_words=20, bits_init=s1["bits"], **cs)
    assert np.array_equal(s2["state"], full["state"])
    assert np.array_equal(s2["bits"][:, :20], full["bits"][:, :20])
    assert np.array_equal(s1["c1"].astype(np.int64) + s2["c1"], full["c1"])


def edge_models():
    rng = np.random.default_rng(0)
    yield "n1_identity", model_from_lists(1, 0.3, [[([0], [0, 1], 1.0)]]), Predicate(
        np.array([0], np.uint16), np.array([1], np.uint8))
    yield "n5_ragged_quads", random_pbn(5, 1, 3, 0, 4, 0.05, seed=1), Predicate(
        np.array([4], np.uint16), np.array([0], np.uint8))
    yield "wide_ell_8", random_pbn(40, 5, 8, 1, 4, 0.01, seed=2), Predicate(
        np.array([0, 39], np.uint16), np.array([1, 1], np.uint8))
    yield "deep_theta_10", random_pbn(64, 1, 3, 6, 10, 0.002, seed=3), Predicate(
        np.array([1, 2, 3], np.uint16), np.array([0, 1, 0], np.uint8))
    yield "theta_7_fast", random_pbn(48, 1, 4, 4, 7, 0.004, seed=6), Predicate(
        np.array([5, 6], np.uint16), np.array([1, 0], np.uint8))
    yield "theta_8_fast", random_pbn(61, 2, 4, 6, 8, 0.004, seed=7), Predicate(
        np.array([60], np.uint16), np.array([1], np.uint8))
    yield "const_functions", random_pbn(37, 1, 4, 0, 1, 0.02, seed=4), Predicate(
        np.zeros(0, np.uint16), np.zeros(0, np.uint8))
    yield "heavy_perturbation", random_pbn(70, 1, 3, 1, 5, 0.3, seed=5), Predicate(
        np.array([69], np.uint16), np.array([1], np.uint8))
    nodes = []
    for i in range(33):
        nodes.append([([int(x) for x in rng.choice(33, 3, replace=False)],
                       [int(b) for b in rng.integers(0, 2, 8)], 1.0)])
    yield "boolean_network_ell1", model_from_lists(33, 1e-3, nodes), Predicate(
        np.array([0], np.uint16), np.array([1], np.uint8))


@pytest.mark.parametrize("cluster_size", [1, 0])
@pytest.mark.parametrize("per_node", [False, True])
@pytest.mark.parametrize("name,model,pred", list(edge_models()), ids=[e[0] for e in edge_models()])
def test_edge_models(pbn, name, model, pred, per_node, cluster_size):
    """cluster_size=1: the single-CTA kernel K1 with the image in shared
    memory (FT = 3..8 and the generic path); 0: auto (45 chains = 2 groups
    -> the cluster kernel wherever the model has enough quads)."""
    full_compare(pbn, model, pred, n_chains=45, steps=777, burn_in=123, seed=17, batch=50,
                 per_node=per_node, cluster_size=cluster_size)


def test_edge_sizes(pbn):
    model, pred = config_model("C1"), config_predicate("C1")
    # steps = 0 (burn-in only), one chain, batch larger than the window
    full_compare(pbn, model, pred, n_chains=1, steps=0, burn_in=50, seed=3)
    full_compare(pbn, model, pred, n_chains=1, steps=1, burn_in=0, seed=3, batch=7)
    full_compare(pbn, model, pred, n_chains=3, steps=31, burn_in=1, seed=3, batch=100)
    full_compare(pbn, model, pred, n_chains=64, steps=33, burn_in=0, seed=3, batch=32)


def test_recount_matches_oracle_subwindows(pbn):
    import torch
    model, pred = config_model("C2"), config_predicate("C2")
    pm = load(pbn, model)
    steps = 1500
    g = gpu_run(pm, model, pred, n_chains=70, steps=steps, burn_in=10, seed=4)
    _, I, _ = oracle_run(model, pred, np.arange(70), steps=steps, burn_in=10, seed=4)
    bits = torch.from_numpy(g["bits"].view(np.int32)).cuda()
    row = g["bits"].shape[1]
    for start, length, batch in [(0, steps, 100), (37, 1000, 33), (1400, 100, 7), (5, 0, 0), (64, 1, 1)]:
        c1 = torch.empty(70, dtype=torch.int32, device="cuda")
        n01, n10 = torch.empty_like(c1), torch.empty_like(c1)
        fl = torch.empty(70, dtype=torch.uint8, device="cuda")
        nb = (length + batch - 1) // batch if batch else 0
        bs = torch.empty((70, max(nb, 1)), dtype=torch.int32, device="cuda") if batch else None
        tot = torch.empty(6, dtype=torch.int64, device="cuda")
        pbn.pbn_recount(bits, 70, row, start, length, batch, c1, n01, n10, fl, bs, tot)
        torch.cuda.synchronize()
        ws = [ostats.window_stats(I[c, start:start + length], batch if batch else 1) for c in range(70)]
        assert np.array_equal(c1.cpu().numpy(), [w.c1 for w in ws])
        assert np.array_equal(n01.cpu().numpy(), [w.n01 for w in ws])
        assert np.array_equal(n10.cpu().numpy(), [w.n10 for w in ws])
        if length:
            assert np.array_equal(fl.cpu().numpy(), [w.first | (w.last << 1) for w in ws])
        if batch:
            assert np.array_equal(bs.cpu().numpy()[:, :nb], np.stack([w.batch_sums for w in ws]))
        assert np.array_equal(tot.cpu().numpy().view(np.uint64), ostats.totals(ws))


def random_props(model, q, rng, kmax=4):
    out = []
    for _ in range(q):
        k = int(rng.integers(0, kmax + 1))
        nodes = rng.choice(model.n, size=k, replace=False).astype(np.uint16)
        out.append(Predicate(nodes, rng.integers(0, 2, size=k).astype(np.uint8)))
    return out


FIELDS = ["c1", "n01", "n10", "first_last", "batch_sums", "bits", "totals"]


@pytest.mark.parametrize("key,q,chains,steps,burn_in,schedule", [
    ("C1", 8, 45, 700, 100, 0),      # n = 10: 3 quads, 8 statistics warps
    ("C2", 5, 200, 600, 150, 0),
    ("C2", 3, 20000, 120, 40, 2),    # persistent chunks carry every property's counters
])
def test_multi_property_equals_single_property_runs(pbn, key, q, chains, steps, burn_in, schedule):
    """q properties abstracted from the same trajectories in one
    launch give exactly the q single-property results."""
    model = config_model(key)
    rng = np.random.default_rng(q)
    props = random_props(model, q, rng)
    pm = load(pbn, model)
    m = gpu_run(pm, model, None, n_chains=chains, steps=steps, burn_in=burn_in, seed=11, batch=64,
                props=props, schedule=schedule, chunk_steps=37 if schedule == 2 else 0)
    for p, pr in enumerate(props):
        s = gpu_run(pm, model, pr, n_chains=chains, steps=steps, burn_in=burn_in, seed=11, batch=64)
        assert np.array_equal(m["state"], s["state"])
        for k in FIELDS:
            assert np.array_equal(m[k][p], s[k]), (p, k)
    # and one property against the oracle on a few chains
    ids = sample_chain_ids(chains, k=4, seed=q)
    st, I, ws = oracle_run(model, props[-1], ids, steps=steps, burn_in=burn_in, seed=11, batch=64)
    packed = pack_states(st)
    last = {k: (m[k][q - 1] if k != "state" else m[k]) for k in ["state"] + FIELDS}
    for j, cid in enumerate(ids):
        compare_chain(last, cid, packed[j], ws[j], steps, 64)


@pytest.mark.parametrize("key,K,chains,per_node", [
    ("C1", 2, 45, False), ("C1", 2, 45, True),
    ("C2", 2, 70, False), ("C2", 4, 33, True), ("C2", 8, 100, False), ("C2", 16, 64, False),
])
def test_cluster_kernel_equals_single_cta(pbn, key, K, chains, per_node):
    """The cluster kernel (one group per K-CTA cluster, state mirrored through
    distributed shared memory) gives exactly the single-CTA kernel's outputs:
    launch-shape independence (A12) across the two kernels."""
    model = config_model(key)
    props = random_props(model, 3, np.random.default_rng(K))
    pm = load(pbn, model, per_node)
    kw = dict(n_chains=chains, steps=333, burn_in=77, seed=5, batch=40, props=props)
    a = gpu_run(pm, model, None, cluster_size=1, **kw)
    b = gpu_run(pm, model, None, cluster_size=K, **kw)
    for k in ["state"] + FIELDS:
        assert np.array_equal(a[k], b[k]), k


def test_cluster_kernel_continuation_and_oracle(pbn):
    """Cluster launches continue chains exactly (init=False, step0 > 0) and
    match the oracle on every chain."""
    model, pred = config_model("C2"), config_predicate("C2")
    pm = load(pbn, model)
    s1 = gpu_run(pm, model, pred, n_chains=40, steps=200, seed=8, cluster_size=4)
    s2 = gpu_run(pm, model, pred, n_chains=40, steps=250, step0=200, seed=8, init=False, state=s1["state"],
                 batch=25, cluster_size=8)
    st, I, ws = oracle_run(model, pred, np.arange(40), steps=450, seed=8)
    packed = pack_states(st)
    assert np.array_equal(s2["state"], packed)
    _, I2, ws2 = oracle_run(model, pred, np.arange(40), steps=250, step0=200, seed=8, batch=25, init=False,
                            state=unpack_states(s1["state"], model.n))
    for c in range(40):
        compare_chain(s2, c, packed[c], ws2[c], 250, 25)


@pytest.mark.parametrize("key,per_node", [("C1", False), ("C2", False), ("C2", True)])
def test_global_image_kernel_small_models(pbn, key, per_node, monkeypatch):
    """The K1 variant that reads the image through L1/L2 (used when the image
    exceeds shared memory, C5) on small models, forced by the test knob
    PBN_FORCE_GLOBAL_IMAGE: identical to the shared-memory kernel and to the
    oracle."""
    model, pred = config_model(key), config_predicate(key)
    pm = load(pbn, model, per_node)
    kw = dict(n_chains=70, steps=400, burn_in=50, seed=21, batch=32, cluster_size=1)
    a = gpu_run(pm, model, pred, **kw)
    monkeypatch.setenv("PBN_FORCE_GLOBAL_IMAGE", "1")
    b = gpu_run(pm, model, pred, **kw)
    monkeypatch.delenv("PBN_FORCE_GLOBAL_IMAGE")
    for k in ["state"] + FIELDS:
        assert np.array_equal(a[k], b[k]), k
    st, I, ws = oracle_run(model, pred, np.arange(70), steps=400, burn_in=50, seed=21, batch=32,
                           per_node=per_node)
    packed = pack_states(st)
    for c in range(70):
        compare_chain(b, c, packed[c], ws[c], 400, 32)


def test_maximum_sizes(pbn):
    """Largest networks and functions this build accepts: n = PBN_MAX_NODES
    (16383, state near the shared-memory limit, image through L1/L2), theta =
    PBN_MAX_THETA (16, generic path) and ell well above the fast path."""
    big = random_pbn(16383, 1, 2, 0, 2, 1e-3, seed=11)
    pred = Predicate(np.array([0, 16382], np.uint16), np.array([1, 0], np.uint8))
    pm = load(pbn, big)
    g = gpu_run(pm, big, pred, n_chains=40, steps=30, burn_in=5, seed=2, batch=7)
    ids = [0, 31, 39]
    st, I, ws = oracle_run(big, pred, ids, steps=30, burn_in=5, seed=2, batch=7)
    packed = pack_states(st)
    for k, c in enumerate(ids):
        compare_chain(g, c, packed[k], ws[k], 30, 7)
    wide = random_pbn(17, 3, 6, 15, 16, 0.01, seed=12)
    pred = Predicate(np.array([3], np.uint16), np.array([1], np.uint8))
    full_compare(pbn, wide, pred, n_chains=35, steps=200, burn_in=20, seed=4, batch=30)


@pytest.mark.parametrize("p", [2.0 ** -32, 0.9])
def test_extreme_perturbation_probabilities(pbn, p):
    """T_p = floor(p 2^32) at its smallest non-zero value (p = 2^-32) and a
    perturbation-dominated chain (p = 0.9), both semantics."""
    model = random_pbn(45, 1, 4, 1, 6, p, seed=13)
    pred = Predicate(np.array([0, 1], np.uint16), np.array([1, 1], np.uint8))
    for per_node in (False, True):
        full_compare(pbn, model, pred, n_chains=40, steps=300, burn_in=10, seed=6, batch=25, per_node=per_node)


# --------------------------------------------------------------------------
# K1n: lanes over nodes, one chain per cluster of K CTAs (pbn_nodepar.cu)
# --------------------------------------------------------------------------
NODE_LANES = 2


@pytest.mark.parametrize("K,G", [(1, 1), (2, 1), (4, 1), (1, 2), (2, 3), (4, 32), (1, 0)])
@pytest.mark.parametrize("per_node", [False, True])
def test_node_lanes_kernel_equals_chain_lanes_and_oracle(pbn, K, G, per_node):
    """The lanes-over-nodes kernel gives exactly the chain-lanes kernel's
    outputs (A12: launch-shape independence across layouts) for every
    cluster size K and chains per cluster G (37 chains: a ragged last
    cluster), with several properties, and matches the oracle."""
    model = config_model("C2")
    props = random_props(model, 3, np.random.default_rng(K + 10 * per_node + 100 * G))
    pm = load(pbn, model, per_node)
    kw = dict(n_chains=37, steps=444, burn_in=55, seed=12, batch=40, props=props)
    a = gpu_run(pm, model, None, cluster_size=1, layout=1, **kw)
    b = gpu_run(pm, model, None, cluster_size=K, layout=NODE_LANES, chains_per_cluster=G, **kw)
    for k in ["state"] + FIELDS:
        assert np.array_equal(a[k], b[k]), (K, G, k)
    ids = [0, 1, 2, 35, 36]
    st, I, ws = oracle_run(model, props[0], ids, steps=444, burn_in=55, seed=12, batch=40, per_node=per_node)
    packed = pack_states(st)
    first = {k: (b[k][0] if k != "state" else b[k]) for k in ["state"] + FIELDS}
    for j, c in enumerate(ids):
        compare_chain(first, c, packed[j], ws[j], 444, 40)


@pytest.mark.parametrize("per_node", [False, True])
@pytest.mark.parametrize("name,model,pred", list(edge_models()), ids=[e[0] for e in edge_models()])
def test_node_lanes_edge_models(pbn, name, model, pred, per_node):
    """Every fast width FT = 3..8, the generic (slow) path, ragged quads,
    n = 1, constant functions, heavy perturbation -- lanes over nodes vs the
    oracle on every chain."""
    pm = load(pbn, model, per_node)
    g = gpu_run(pm, model, pred, n_chains=6, steps=555, burn_in=77, seed=19, batch=50, layout=NODE_LANES)
    st, I, ws = oracle_run(model, pred, np.arange(6), steps=555, burn_in=77, seed=19, batch=50, per_node=per_node)
    packed = pack_states(st)
    for c in range(6):
        compare_chain(g, c, packed[c], ws[c], 555, 50)
    assert np.array_equal(g["totals"], ostats.totals(ws))


def test_node_lanes_continuation_and_chain_base(pbn):
    """Chains continue exactly across calls and layouts (init=False, step0 > 0,
    chain_base > 0, bits appended at an offset)."""
    model, pred = config_model("C3"), config_predicate("C3")
    pm = load(pbn, model)
    s1 = gpu_run(pm, model, pred, n_chains=3, chain_base=40, steps=300, seed=8, layout=NODE_LANES,
                 bits_row_words=30)
    s2 = gpu_run(pm, model, pred, n_chains=3, chain_base=40, steps=500, step0=300, seed=8, init=False,
                 state=s1["state"], batch=25, layout=NODE_LANES, cluster_size=4, bits_offset=300, bits_row_words=30,
                 bits_init=s1["bits"])
    full = gpu_run(pm, model, pred, n_chains=3, chain_base=40, steps=800, seed=8, layout=1, cluster_size=1)
    assert np.array_equal(s2["state"], full["state"])
    assert np.array_equal(s2["bits"][:, :25], full["bits"][:, :25])
    st, I, ws = oracle_run(model, pred, [40, 41, 42], steps=800, seed=8)
    assert np.array_equal(s2["state"], pack_states(st))


@pytest.mark.parametrize("K", [8, 16])
def test_node_lanes_C5(pbn, K):
    """C5 (n = 5000, image 871 KB: sub-images of 1/8 or 1/16 per CTA) with
    lanes over nodes: 1 and 3 chains at the sweep's 10^4 steps vs the oracle."""
    c = CONFIGS["C5"]
    model, pred = config_model("C5"), config_predicate("C5")
    pm = load(pbn, model)
    for chains, G in ((1, 1), (3, 1), (5, 2)):
        g = gpu_run(pm, model, pred, n_chains=chains, steps=c.steps, burn_in=c.burn_in, seed=c.sim_seed,
                    batch=c.batch, layout=NODE_LANES, cluster_size=K, chains_per_cluster=G)
        st, I, ws = oracle_run(model, pred, np.arange(chains), steps=c.steps, burn_in=c.burn_in, seed=c.sim_seed,
                               batch=c.batch, threads=os.cpu_count() or 8)
        packed = pack_states(st)
        for j in range(chains):
            compare_chain(g, j, packed[j], ws[j], c.steps, c.batch)


# --------------------------------------------------------------------------
# NEXT-3: the dense class (density 150-300): the generic path
# with binary-search selection and warp-uniform gathers
# --------------------------------------------------------------------------
def test_dense_class_C6_sampled_chains(pbn):
    """C6 (n = 1000, ell ~ U{8..24}, theta ~ U{8..12}, density ~160; image
    ~5 MB read through L1/L2) in bench.py's launch configuration, 32 sampled
    chains against the oracle at the full step count, invariants on all."""
    c = CONFIGS["C6"]
    model, pred = config_model("C6"), config_predicate("C6")
    pm = load(pbn, model)
    g = gpu_run(pm, model, pred, n_chains=c.chains, steps=c.steps, burn_in=c.burn_in, seed=c.sim_seed, batch=c.batch)
    ids = sample_chain_ids(c.chains, k=32, seed=c.sim_seed)
    st, I, ws = oracle_run(model, pred, ids, steps=c.steps, burn_in=c.burn_in, seed=c.sim_seed, batch=c.batch,
                           threads=os.cpu_count() or 8)
    packed = pack_states(st)
    for k, cid in enumerate(ids):
        compare_chain(g, cid, packed[k], ws[k], c.steps, c.batch)
    c1 = g["c1"].astype(np.int64)
    assert np.array_equal(g["batch_sums"].astype(np.int64).sum(axis=1), c1)
    assert np.array_equal(np.unpackbits(g["bits"].view(np.uint8), axis=1).sum(axis=1), c1)


@pytest.mark.parametrize("per_node", [False, True])
def test_dense_small_model_every_kernel(pbn, per_node, monkeypatch):
    """A small dense model (ell up to 20, theta 8..11) through K1 with the
    image in shared memory, K1 reading it through L1/L2, the cluster kernel
    and lanes over nodes -- all against the oracle on every chain."""
    model = random_pbn(70, 5, 20, 8, 11, 0.003, seed=31)
    pred = Predicate(np.array([0, 69], np.uint16), np.array([1, 0], np.uint8))
    pm = load(pbn, model, per_node)
    kw = dict(n_chains=40, steps=500, burn_in=40, seed=5, batch=25)
    st, I, ws = oracle_run(model, pred, np.arange(40), steps=500, burn_in=40, seed=5, batch=25, per_node=per_node)
    packed = pack_states(st)
    runs = {"K1 smem": dict(cluster_size=1), "K1c K=2": dict(cluster_size=2), "K1n": dict(layout=NODE_LANES)}
    for name, extra in runs.items():
        try:
            g = gpu_run(pm, model, pred, **kw, **extra)
        except Exception as e:  # a layout whose image does not fit shared memory
            assert "USAGE" in str(e), (name, e)
            continue
        for c in range(40):
            compare_chain(g, c, packed[c], ws[c], 500, 25)
    monkeypatch.setenv("PBN_FORCE_GLOBAL_IMAGE", "1")
    g = gpu_run(pm, model, pred, cluster_size=1, **kw)
    monkeypatch.delenv("PBN_FORCE_GLOBAL_IMAGE")
    for c in range(40):
        compare_chain(g, c, packed[c], ws[c], 500, 25)


# --------------------------------------------------------------------------
# NEXT-2: the geometric-skip perturbation stream (PBN_PERTURB_GEOMETRIC,
# reading Q18; oracle pinned in test_oracle_geometric.py)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("key,chains", [("C1", 4), ("C2", 200), ("C3", 64)])
def test_geometric_mode_all_chains(pbn, key, chains):
    c = CONFIGS[key]
    model, pred = config_model(key), config_predicate(key)
    pm = pbn.pbn_load(model, geometric=True)
    steps, burn_in = min(c.steps, 3000), min(c.burn_in, 500)
    g = gpu_run(pm, model, pred, n_chains=chains, steps=steps, burn_in=burn_in, seed=c.sim_seed, batch=c.batch)
    st, I, ws = oracle_run(model, pred, np.arange(chains), steps=steps, burn_in=burn_in, seed=c.sim_seed,
                           batch=c.batch, geometric=True, threads=os.cpu_count() or 8)
    packed = pack_states(st)
    for j in range(chains):
        compare_chain(g, j, packed[j], ws[j], steps, c.batch)
    assert np.array_equal(g["totals"], ostats.totals(ws))


def test_geometric_mode_C4_sampled_chains_and_launch_shapes(pbn):
    """C4 at its full size with the geometric stream (persistent schedule),
    sampled chains vs the oracle; plus launch-shape independence (warps,
    persistent chunks, global image) on a ragged chain count."""
    c = CONFIGS["C4"]
    model, pred = config_model("C4"), config_predicate("C4")
    pm = pbn.pbn_load(model, geometric=True)
    g = gpu_run(pm, model, pred, n_chains=c.chains, steps=c.steps, burn_in=c.burn_in, seed=c.sim_seed, batch=c.batch)
    ids = sample_chain_ids(c.chains, k=24, seed=c.sim_seed)
    st, I, ws = oracle_run(model, pred, ids, steps=c.steps, burn_in=c.burn_in, seed=c.sim_seed, batch=c.batch,
                           geometric=True, threads=os.cpu_count() or 8)
    packed = pack_states(st)
    for k, cid in enumerate(ids):
        compare_chain(g, cid, packed[k], ws[k], c.steps, c.batch)
    kw = dict(n_chains=1000, steps=300, burn_in=40, seed=3, batch=30)
    ref = gpu_run(pm, model, pred, schedule=1, **kw)
    for extra in [dict(warps=7, schedule=1), dict(schedule=2, chunk_steps=17), dict(schedule=0)]:
        b = gpu_run(pm, model, pred, **kw, **extra)
        for k in ALL:
            assert np.array_equal(ref[k], b[k]), (extra, k)
    import os as _os
    _os.environ["PBN_FORCE_GLOBAL_IMAGE"] = "1"
    try:
        b = gpu_run(pm, model, pred, schedule=1, **kw)
    finally:
        del _os.environ["PBN_FORCE_GLOBAL_IMAGE"]
    for k in ALL:
        assert np.array_equal(ref[k], b[k]), ("global image", k)


def test_geometric_mode_rejects_the_cluster_kernel(pbn):
    import paper_1508_07828_b200 as P
    model, pred = config_model("C2"), config_predicate("C2")
    pm = pbn.pbn_load(model, geometric=True)
    with pytest.raises(P.PbnError):
        gpu_run(pm, model, pred, n_chains=40, steps=10, cluster_size=2)


@pytest.mark.parametrize("key,K,G", [("C1", 1, 1), ("C2", 2, 3), ("C3", 4, 2), ("C5", 8, 2)])
def test_geometric_mode_node_lanes(pbn, key, K, G):
    """Lanes over nodes with the geometric stream (chain-steps with gamma != 0
    skip the evaluation): identical to K1 and to the oracle."""
    c = CONFIGS[key]
    model, pred = config_model(key), config_predicate(key)
    pm = pbn.pbn_load(model, geometric=True)
    chains = 5
    steps, burn_in = min(c.steps, 2000), min(c.burn_in, 300)
    kw = dict(n_chains=chains, steps=steps, burn_in=burn_in, seed=c.sim_seed, batch=c.batch)
    a = gpu_run(pm, model, pred, cluster_size=1, layout=1, **kw)
    b = gpu_run(pm, model, pred, cluster_size=K, layout=NODE_LANES, chains_per_cluster=G, **kw)
    for k in ALL:
        assert np.array_equal(a[k], b[k]), k
    st, I, ws = oracle_run(model, pred, np.arange(chains), steps=steps, burn_in=burn_in, seed=c.sim_seed,
                           batch=c.batch, geometric=True, threads=os.cpu_count() or 8)
    packed = pack_states(st)
    for j in range(chains):
        compare_chain(b, j, packed[j], ws[j], steps, c.batch)
