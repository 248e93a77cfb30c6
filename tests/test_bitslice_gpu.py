"""GPU parity of K1b, the bit-sliced evaluation kernel (layout
PBN_LAYOUT_BITSLICE = 3): bit-exact against the CPU oracle on every output
field, and bit-identical to K1 (cluster_size=1) across launch shapes --
BASELINE north_star ("GPU trajectories, counts and transition tallies must be
bit-exact against the oracle"); the step it computes is PAPER P:132-167 and
the semantics P:159-165 (VECTOR) / reading Q1 (PER_NODE)."""
import os

import numpy as np
import pytest

from tests.helpers import compare_chain, gpu_run, oracle_run, pack_states, sample_chain_ids
from oracle import stats as ostats
from workloads import CONFIGS, Predicate, config_model, config_predicate, model_from_lists, random_pbn

pytestmark = pytest.mark.gpu
BS = 3  # PBN_LAYOUT_BITSLICE
ALL = ["state", "c1", "n01", "n10", "first_last", "batch_sums", "bits", "totals"]


@pytest.fixture(scope="module")
def pbn():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1508_07828_b200 as pbn
    return pbn


def full_compare(pbn, model, pred, *, n_chains, steps, burn_in=0, seed=1, batch=0, per_node=False, **kw):
    pm = pbn.pbn_load(model, per_node=per_node)
    g = gpu_run(pm, model, pred, n_chains=n_chains, steps=steps, burn_in=burn_in, seed=seed, batch=batch,
                layout=BS, **kw)
    st, I, ws = oracle_run(model, pred, np.arange(n_chains), steps=steps, burn_in=burn_in, seed=seed,
                           batch=batch, per_node=per_node, threads=8)
    packed = pack_states(st)
    for c in range(n_chains):
        compare_chain(g, c, packed[c], ws[c], steps, batch)
    assert np.array_equal(g["totals"], ostats.totals(ws))
    return g


@pytest.mark.parametrize("per_node", [False, True])
@pytest.mark.parametrize("key", ["C1", "C2"])
def test_small_configs_all_chains(pbn, key, per_node):
    c = CONFIGS[key]
    full_compare(pbn, config_model(key), config_predicate(key), n_chains=c.chains, steps=c.steps,
                 burn_in=c.burn_in, seed=c.sim_seed, batch=c.batch, per_node=per_node)


def bs_models():
    """Models inside K1b's shape (theta <= 6, ell <= 4): every class 1..6,
    ragged quads, constant functions, one function per node, heavy p."""
    rng = np.random.default_rng(0)
    yield "n1_identity", model_from_lists(1, 0.3, [[([0], [0, 1], 1.0)]]), Predicate(
        np.array([0], np.uint16), np.array([1], np.uint8))
    yield "n5_ragged_quads", random_pbn(5, 1, 3, 0, 4, 0.05, seed=1), Predicate(
        np.array([4], np.uint16), np.array([0], np.uint8))
    yield "n7_ell4_theta6", random_pbn(7, 4, 4, 6, 6, 0.01, seed=11), Predicate(
        np.array([6], np.uint16), np.array([1], np.uint8))
    yield "n150_all_classes", random_pbn(150, 1, 4, 0, 6, 0.003, seed=12), Predicate(
        np.array([0, 149, 77], np.uint16), np.array([1, 0, 1], np.uint8))
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
    yield "theta_7_classes", random_pbn(48, 1, 4, 4, 7, 0.004, seed=6), Predicate(
        np.array([5, 6], np.uint16), np.array([1, 0], np.uint8))
    yield "theta_8_classes", random_pbn(61, 2, 4, 6, 8, 0.004, seed=7), Predicate(
        np.array([60], np.uint16), np.array([1], np.uint8))
    yield "ell3_theta1_8", random_pbn(130, 1, 3, 1, 8, 0.002, seed=13), Predicate(
        np.array([3, 129], np.uint16), np.array([0, 1], np.uint8))


@pytest.mark.parametrize("per_node", [False, True])
@pytest.mark.parametrize("name,model,pred", list(bs_models()), ids=[e[0] for e in bs_models()])
def test_models_all_chains(pbn, name, model, pred, per_node):
    full_compare(pbn, model, pred, n_chains=45, steps=777, burn_in=123, seed=17, batch=50, per_node=per_node)


@pytest.mark.parametrize("per_node", [False, True])
@pytest.mark.parametrize("name", ["n150_all_classes", "theta_8_classes", "ell3_theta1_8"])
def test_models_global_image(pbn, name, per_node, monkeypatch):
    """The image read through L1/L2 instead of staged (the C5 shape):
    PBN_FORCE_GLOBAL_IMAGE=1 forces it for small models."""
    model, pred = {k: (m, p) for k, m, p in bs_models()}[name]
    monkeypatch.setenv("PBN_FORCE_GLOBAL_IMAGE", "1")
    full_compare(pbn, model, pred, n_chains=70, steps=555, burn_in=45, seed=23, batch=37, per_node=per_node)
    assert pbn.pbn_last_kernel() == "K1b-global"


@pytest.mark.parametrize("per_node", [False, True])
def test_launch_shapes_equal_K1(pbn, per_node):
    """Warps per group 1..24 and persistent chunks straddling the burn-in
    end, batch and bit-word boundaries give K1's outputs exactly."""
    model, pred = config_model("C2"), config_predicate("C2")
    pm = pbn.pbn_load(model, per_node=per_node)
    kw = dict(n_chains=200, steps=700, burn_in=300, seed=9, batch=64)
    ref = gpu_run(pm, model, pred, cluster_size=1, schedule=1, **kw)
    for warps in [0, 1, 2, 5, 7, 8, 13, 20, 21, 24]:  # (<= 20: the 640-thread build; 24 = K1b's warp budget)
        g = gpu_run(pm, model, pred, warps=warps, schedule=1, layout=BS, **kw)
        for k in ALL:
            assert np.array_equal(g[k], ref[k]), (warps, k)
    for chunk, warps in [(1, 4), (7, 24), (33, 3), (299, 0), (1000, 8), (0, 0)]:
        g = gpu_run(pm, model, pred, warps=warps, schedule=2, chunk_steps=chunk, layout=BS, **kw)
        for k in ALL:
            assert np.array_equal(g[k], ref[k]), ("persistent", chunk, warps, k)


@pytest.mark.parametrize("per_node", [False, True])
def test_ragged_group_persistent(pbn, per_node):
    """20007 chains (7 real lanes in the last group), persistent with short
    chunks: equal to the one-CTA-per-group launch and to the oracle."""
    model, pred = config_model("C2"), config_predicate("C2")
    pm = pbn.pbn_load(model, per_node=per_node)
    kw = dict(n_chains=20007, steps=300, burn_in=60, seed=4, batch=50, layout=BS)
    a = gpu_run(pm, model, pred, schedule=1, **kw)
    b = gpu_run(pm, model, pred, schedule=2, chunk_steps=13, **kw)
    for k in ALL:
        assert np.array_equal(a[k], b[k]), k
    ids = [0, 19999, 20000, 20006] + sample_chain_ids(20007, k=4, seed=2)
    st, I, ws = oracle_run(model, pred, ids, steps=300, burn_in=60, seed=4, batch=50, per_node=per_node)
    packed = pack_states(st)
    for j, cid in enumerate(ids):
        compare_chain(b, cid, packed[j], ws[j], 300, 50)


def test_chain_split_and_step_split(pbn):
    model, pred = config_model("C2"), config_predicate("C2")
    pm = pbn.pbn_load(model)
    full = gpu_run(pm, model, pred, n_chains=100, steps=640, seed=5, layout=BS)
    a = gpu_run(pm, model, pred, n_chains=37, steps=640, seed=5, layout=BS)
    b = gpu_run(pm, model, pred, n_chains=63, chain_base=37, steps=640, seed=5, layout=BS)
    for k in ["state", "c1", "n01", "n10", "first_last", "bits"]:
        assert np.array_equal(np.concatenate([a[k], b[k]]), full[k]), k
    s1 = gpu_run(pm, model, pred, n_chains=100, steps=300, seed=5, bits_row_words=20, layout=BS)
    s2 = gpu_run(pm, model, pred, n_chains=100, steps=340, step0=300, seed=5, init=False, state=s1["state"],
                 bits_offset=300, bits_row_words=20, bits_init=s1["bits"], layout=BS)
    assert np.array_equal(s2["state"], full["state"])
    assert np.array_equal(s2["bits"][:, :20], full["bits"][:, :20])
    assert np.array_equal(s1["c1"].astype(np.int64) + s2["c1"], full["c1"])


def test_multi_property(pbn):
    model = config_model("C2")
    rng = np.random.default_rng(3)
    props = []
    for _ in range(5):
        k = int(rng.integers(0, 5))
        props.append(Predicate(rng.choice(model.n, size=k, replace=False).astype(np.uint16),
                               rng.integers(0, 2, size=k).astype(np.uint8)))
    pm = pbn.pbn_load(model)
    kw = dict(n_chains=200, steps=600, burn_in=150, seed=11, batch=64, props=props)
    a = gpu_run(pm, model, None, cluster_size=1, **kw)
    b = gpu_run(pm, model, None, layout=BS, **kw)
    for k in ALL:
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("key", ["C3", "C4"])
def test_large_configs_sampled_chains(pbn, key):
    """The full C3 / C4 launch (auto: K1b, the bench shape); the oracle
    recomputes 64 sampled chains at the full step count; invariants on every
    chain."""
    c = CONFIGS[key]
    model, pred = config_model(key), config_predicate(key)
    pm = pbn.pbn_load(model)
    # auto layout: the kernel bench.py times on these configs
    g = gpu_run(pm, model, pred, n_chains=c.chains, steps=c.steps, burn_in=c.burn_in, seed=c.sim_seed,
                batch=c.batch)
    assert pbn.pbn_last_kernel() == "K1b"
    ids = sample_chain_ids(c.chains, k=64, seed=c.sim_seed)
    st, I, ws = oracle_run(model, pred, ids, steps=c.steps, burn_in=c.burn_in, seed=c.sim_seed, batch=c.batch,
                           threads=os.cpu_count() or 8)
    packed = pack_states(st)
    for k, cid in enumerate(ids):
        compare_chain(g, cid, packed[k], ws[k], c.steps, c.batch)
    c1 = g["c1"].astype(np.int64)
    fl = g["first_last"].astype(np.int64)
    first, last = fl & 1, fl >> 1
    assert np.array_equal(g["n01"].astype(np.int64) - g["n10"].astype(np.int64), last - first)
    assert np.array_equal(g["batch_sums"].astype(np.int64).sum(axis=1), c1)
    assert np.array_equal(np.unpackbits(g["bits"].view(np.uint8), axis=1).sum(axis=1), c1)


def test_outside_shape_is_refused(pbn):
    """theta > 8 (or ell > 4, or the geometric stream) has no K1b image: the
    forced layout fails loudly instead of falling back."""
    model = random_pbn(64, 1, 3, 6, 10, 0.002, seed=3)
    pm = pbn.pbn_load(model)
    with pytest.raises(Exception):
        gpu_run(pm, model, Predicate(np.array([5], np.uint16), np.array([1], np.uint8)), n_chains=40, steps=10,
                layout=BS)


# NEXT-2 in K1b: the geometric-skip stream (reading Q18; oracle pinned in
# tests/test_oracle_geometric.py): one warp per step clears the gamma words
# and draws gamma(t) by skips, every other step part as VECTOR
@pytest.mark.parametrize("key,chains", [("C1", 4), ("C2", 200), ("C3", 64)])
def test_geometric_all_chains(pbn, key, chains):
    c = CONFIGS[key]
    model, pred = config_model(key), config_predicate(key)
    pm = pbn.pbn_load(model, geometric=True)
    steps, burn_in = min(c.steps, 3000), min(c.burn_in, 500)
    g = gpu_run(pm, model, pred, n_chains=chains, steps=steps, burn_in=burn_in, seed=c.sim_seed, batch=c.batch,
                layout=BS)
    assert pbn.pbn_last_kernel() == "K1b"
    st, I, ws = oracle_run(model, pred, np.arange(chains), steps=steps, burn_in=burn_in, seed=c.sim_seed,
                           batch=c.batch, geometric=True, threads=os.cpu_count() or 8)
    packed = pack_states(st)
    for j in range(chains):
        compare_chain(g, j, packed[j], ws[j], steps, c.batch)
    assert np.array_equal(g["totals"], ostats.totals(ws))


def test_geometric_launch_shapes_equal_K1(pbn, monkeypatch):
    """Warps, persistent chunks, a ragged group and the global image give K1's
    outputs exactly under the geometric stream."""
    model, pred = config_model("C2"), config_predicate("C2")
    pm = pbn.pbn_load(model, geometric=True)
    kw = dict(n_chains=2007, steps=400, burn_in=90, seed=6, batch=40)
    ref = gpu_run(pm, model, pred, cluster_size=1, layout=1, schedule=1, **kw)
    assert pbn.pbn_last_kernel() == "K1"
    for extra in [dict(warps=1), dict(warps=9), dict(warps=0, schedule=2, chunk_steps=13),
                  dict(warps=24, schedule=2, chunk_steps=1)]:
        g = gpu_run(pm, model, pred, layout=BS, **kw, **extra)
        for k in ALL:
            assert np.array_equal(g[k], ref[k]), (extra, k)
    monkeypatch.setenv("PBN_FORCE_GLOBAL_IMAGE", "1")
    g = gpu_run(pm, model, pred, layout=BS, **kw)
    assert pbn.pbn_last_kernel() == "K1b-global"
    for k in ALL:
        assert np.array_equal(g[k], ref[k]), ("global image", k)


# K1bc: one 32-chain group per cluster of K CTAs (each owns a slice of the
# quads and its sub-image; new words and any words exchanged through
# distributed shared memory every step)
@pytest.mark.parametrize("per_node", [False, True])
@pytest.mark.parametrize("K", [2, 4, 8, 16])
def test_cluster_equals_K1_and_oracle(pbn, K, per_node):
    model, pred = config_model("C2"), config_predicate("C2")
    pm = pbn.pbn_load(model, per_node=per_node)
    kw = dict(n_chains=100, steps=500, burn_in=120, seed=12, batch=45)
    ref = gpu_run(pm, model, pred, cluster_size=1, layout=1, schedule=1, **kw)
    g = gpu_run(pm, model, pred, cluster_size=K, layout=BS, **kw)
    assert pbn.pbn_last_kernel() == "K1bc"
    for k in ALL:
        assert np.array_equal(g[k], ref[k]), (K, k)
    ids = sample_chain_ids(100, k=6, seed=K)
    st, I, ws = oracle_run(model, pred, ids, steps=500, burn_in=120, seed=12, batch=45, per_node=per_node)
    packed = pack_states(st)
    for j, cid in enumerate(ids):
        compare_chain(g, cid, packed[j], ws[j], 500, 45)


@pytest.mark.parametrize("name,K", [("n5_ragged_quads", 2), ("n150_all_classes", 4), ("theta_8_classes", 2),
                                    ("ell3_theta1_8", 8), ("heavy_perturbation", 4)])
def test_cluster_models(pbn, name, K):
    model, pred = {k: (m, p) for k, m, p in bs_models()}[name]
    pm = pbn.pbn_load(model)
    kw = dict(n_chains=45, steps=600, burn_in=77, seed=31, batch=40)
    g = gpu_run(pm, model, pred, cluster_size=K, layout=BS, **kw)
    assert pbn.pbn_last_kernel() == "K1bc"
    st, I, ws = oracle_run(model, pred, np.arange(45), steps=600, burn_in=77, seed=31, batch=40)
    packed = pack_states(st)
    for c in range(45):
        compare_chain(g, c, packed[c], ws[c], 600, 40)
    assert np.array_equal(g["totals"], ostats.totals(ws))


def test_cluster_geometric_and_multi_property(pbn):
    model = config_model("C2")
    rng = np.random.default_rng(5)
    props = []
    for _ in range(3):
        k = int(rng.integers(1, 5))
        props.append(Predicate(rng.choice(model.n, size=k, replace=False).astype(np.uint16),
                               rng.integers(0, 2, size=k).astype(np.uint8)))
    pm = pbn.pbn_load(model, geometric=True)
    kw = dict(n_chains=70, steps=400, burn_in=50, seed=8, batch=25, props=props)
    ref = gpu_run(pm, model, None, cluster_size=1, layout=1, **kw)
    g = gpu_run(pm, model, None, cluster_size=4, layout=BS, **kw)
    for k in ALL:
        assert np.array_equal(g[k], ref[k]), k


def test_cluster_C5_1024_sampled_chains(pbn):
    """C5 at 1024 chains (its sweep point, 32 groups) through K1bc; the
    oracle recomputes sampled chains at the full step count."""
    c = CONFIGS["C5"]
    model, pred = config_model("C5"), config_predicate("C5")
    pm = pbn.pbn_load(model)
    g = gpu_run(pm, model, pred, n_chains=1024, steps=c.steps, burn_in=c.burn_in, seed=c.sim_seed, batch=c.batch,
                cluster_size=4, layout=BS)
    assert pbn.pbn_last_kernel() == "K1bc"
    ids = sample_chain_ids(1024, k=12, seed=c.sim_seed)
    st, I, ws = oracle_run(model, pred, ids, steps=c.steps, burn_in=c.burn_in, seed=c.sim_seed, batch=c.batch,
                           threads=os.cpu_count() or 8)
    packed = pack_states(st)
    for k, cid in enumerate(ids):
        compare_chain(g, cid, packed[k], ws[k], c.steps, c.batch)


@pytest.mark.parametrize("cluster", [1, 2])
def test_edge_sizes(pbn, cluster):
    """Zero recorded steps (burn-in only), one step, a batch longer than the
    window, a ragged group: K1b (cluster 1) and K1bc (cluster 2)."""
    model, pred = config_model("C2"), config_predicate("C2")
    for n_chains, steps, burn_in, batch in [(33, 0, 50, 0), (40, 1, 0, 7), (70, 31, 1, 100), (5, 0, 0, 0)]:
        full_compare(pbn, model, pred, n_chains=n_chains, steps=steps, burn_in=burn_in, seed=3, batch=batch,
                     cluster_size=cluster)
        assert pbn.pbn_last_kernel() == ("K1b" if cluster == 1 else "K1bc")


def test_cluster_continuation_and_chain_split(pbn):
    """K1bc continues chains exactly (init=False, step0 > 0, bits appended at
    an offset) and splits chains across calls (chain_base)."""
    model, pred = config_model("C3"), config_predicate("C3")
    pm = pbn.pbn_load(model)
    kw = dict(cluster_size=4, layout=BS)
    full = gpu_run(pm, model, pred, n_chains=64, steps=480, seed=5, **kw)
    s1 = gpu_run(pm, model, pred, n_chains=64, steps=200, seed=5, bits_row_words=15, **kw)
    s2 = gpu_run(pm, model, pred, n_chains=64, steps=280, step0=200, seed=5, init=False, state=s1["state"],
                 bits_offset=200, bits_row_words=15, bits_init=s1["bits"], **kw)
    assert np.array_equal(s2["state"], full["state"])
    assert np.array_equal(s2["bits"][:, :15], full["bits"][:, :15])
    assert np.array_equal(s1["c1"].astype(np.int64) + s2["c1"], full["c1"])
    a = gpu_run(pm, model, pred, n_chains=37, steps=480, seed=5, **kw)
    b = gpu_run(pm, model, pred, n_chains=27, chain_base=37, steps=480, seed=5, **kw)
    for k in ["state", "c1", "n01", "n10", "first_last", "bits"]:
        assert np.array_equal(np.concatenate([a[k], b[k]]), full[k]), k
