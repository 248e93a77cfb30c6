"""Shared test helpers: run the CUDA path through the C ABI and the oracle on
the same seeded inputs, and compare field by field."""
from __future__ import annotations

import numpy as np

from oracle import sim as osim
from oracle import stats as ostats


def pack_states(st: np.ndarray) -> np.ndarray:
    """[chains x n] 0/1 bytes -> [chains x ceil(n/32)] u32, node i = bit i&31 of word i>>5."""
    chains, n = st.shape
    nw = (n + 31) // 32
    out = np.zeros((chains, nw), np.uint64)
    for i in range(n):
        out[:, i >> 5] |= st[:, i].astype(np.uint64) << np.uint64(i & 31)
    return out.astype(np.uint32)


def unpack_states(words: np.ndarray, n: int) -> np.ndarray:
    w = words.astype(np.uint64)
    return np.stack([((w[:, i >> 5] >> np.uint64(i & 31)) & np.uint64(1)).astype(np.uint8)
                     for i in range(n)], axis=1)


def sample_chain_ids(n_chains: int, k: int = 8, seed: int = 0) -> list[int]:
    """Deterministic subset: ends of the first groups, the last chain and hashed ids."""
    base = [0, 1, 31, 32, n_chains - 1]
    rng = np.random.default_rng(seed)
    extra = [int(x) for x in rng.integers(0, n_chains, size=max(0, k - len(base)))]
    out = []
    for c in base + extra:
        if 0 <= c < n_chains and c not in out:
            out.append(c)
    return out


def gpu_run(pm, model, pred, *, n_chains, steps, burn_in=0, step0=0, chain_base=0, seed=1, batch=0,
            emit_bits=True, init=True, state=None, groups=0, warps=0, bits_offset=0,
            bits_row_words=0, bits_init=None, schedule=0, chunk_steps=0, props=None, cluster_size=0, layout=0,
            chains_per_cluster=0):
    """Run pbn_simulate; returns a dict of host numpy arrays (with `props`,
    every field but state has a leading property dimension)."""
    import torch
    import paper_1508_07828_b200 as pbn
    out = pbn.alloc_outputs(pm, n_chains, steps, batch=batch, emit_bits=emit_bits,
                            bits_row_words=bits_row_words, n_props=len(props) if props else 0)
    if state is not None:
        out.state.copy_(torch.from_numpy(np.ascontiguousarray(state).view(np.int32)).cuda())
    if bits_init is not None:
        out.bits.copy_(torch.from_numpy(np.ascontiguousarray(bits_init).view(np.int32)).cuda())
    pbn.pbn_simulate(pm, out, n_chains=n_chains, steps=steps, chain_base=chain_base, step0=step0,
                     burn_in=burn_in, batch=batch, seed=seed, pred=pred, init=init,
                     emit_bits=emit_bits, bits_offset=bits_offset, bits_row_words=bits_row_words,
                     groups_per_cta=groups, warps_per_group=warps, schedule=schedule,
                     chunk_steps=chunk_steps, props=props, cluster_size=cluster_size, layout=layout,
                     chains_per_cluster=chains_per_cluster)
    torch.cuda.synchronize()

    def h(t):
        return None if t is None else t.cpu().numpy()

    r = {k: h(getattr(out, k)) for k in ["state", "c1", "n01", "n10", "first_last", "batch_sums",
                                         "bits", "totals"]}
    for k in ["state", "c1", "n01", "n10", "batch_sums", "bits"]:
        if r[k] is not None:
            r[k] = r[k].view(np.uint32)
    r["totals"] = r["totals"].view(np.uint64)
    return r


def oracle_run(model, pred, chain_ids, *, steps, burn_in=0, step0=0, seed=1, batch=0, init=True,
               state=None, per_node=False, threads=8, geometric=False):
    st, I = osim.simulate(model, pred, seed=seed, chain_ids=np.asarray(chain_ids, np.uint32),
                          step0=step0, burn_in=burn_in, steps=steps, init=init, state=state,
                          per_node=per_node, threads=threads, geometric=geometric)
    ws = [ostats.window_stats(I[c], batch if batch > 0 else max(steps, 1)) for c in range(len(chain_ids))]
    return st, I, ws


def compare_chain(gpu: dict, row: int, st_packed: np.ndarray, ws, steps: int, batch: int,
                  emit_bits: bool = True):
    """Bit-exact comparison of one chain's every output field."""
    assert np.array_equal(gpu["state"][row], st_packed), f"state row {row}"
    assert int(gpu["c1"][row]) == ws.c1, (row, int(gpu["c1"][row]), ws.c1)
    assert int(gpu["n01"][row]) == ws.n01, row
    assert int(gpu["n10"][row]) == ws.n10, row
    fl = int(gpu["first_last"][row])
    if steps > 0:
        assert fl == (ws.first | (ws.last << 1)), row
    if batch > 0:
        assert np.array_equal(gpu["batch_sums"][row].astype(np.int64), ws.batch_sums), row
    if emit_bits and steps > 0:
        assert np.array_equal(gpu["bits"][row][:len(ws.bits)], ws.bits), row


class GpuChains:
    """Sample source for the oracle drivers (oracle/driver.py) backed by the
    CUDA path: omega chains advanced with pbn_simulate (state carried between
    calls, indicator bits read back).  Lets the oracle's own decision code run
    on GPU trajectories at sizes the oracle simulator cannot reach (C3); the
    trajectories themselves are pinned bit-exact to the oracle on sampled
    chains by test_parity_gpu.py."""

    def __init__(self, pbn, pm, pred, seed: int, omega: int, chain_base: int = 0):
        self.pbn, self.pm, self.pred, self.seed = pbn, pm, pred, seed
        self.omega, self.chain_base = omega, chain_base
        self.length = 0
        self.state = None

    def advance(self, burn_in: int, steps: int) -> np.ndarray:
        import torch
        out = self.pbn.alloc_outputs(self.pm, self.omega, steps, emit_bits=True)
        if self.state is not None:
            out.state.copy_(self.state)
        self.pbn.pbn_simulate(self.pm, out, n_chains=self.omega, chain_base=self.chain_base, steps=steps,
                              step0=self.length, burn_in=burn_in, seed=self.seed, pred=self.pred,
                              init=self.state is None, emit_bits=True)
        torch.cuda.synchronize()
        self.state = out.state.clone()
        self.length += burn_in + steps
        if steps == 0:
            return np.zeros((self.omega, 0), np.uint8)
        bits = np.ascontiguousarray(out.bits.cpu().numpy().view(np.uint32))
        return np.unpackbits(bits.view(np.uint8), axis=1, bitorder="little")[:, :steps]
