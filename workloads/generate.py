"""Seeded PBN generators, the BASELINE.json configs C1-C5 and C6 (dense class).

Layout of a model (CSR, the same arrays `pbn_load` takes, include/pbnsim.h):
  n         number of nodes (V = (v_1..v_n))
  fn_off    int32[n+1]   node i owns functions fn_off[i] .. fn_off[i+1]-1
                         (the set F_i, ell(i) = fn_off[i+1]-fn_off[i] >= 1)
  par_off   int32[nf+1]  function f reads parents[par_off[f] .. par_off[f+1]-1]
  parents   uint16[...]  parent node ids; parents[par_off[f]] is the MOST
                         significant bit of the truth-table index
  tbl_off   int32[nf+1]  function f's table is tables[tbl_off[f] .. tbl_off[f+1]-1]
  tables    uint32[...]  ceil(2^theta/32) words; entry idx is bit (idx & 31)
                         of word idx >> 5 (bit 0 of word 0 = all-parents-zero)
  sel_prob  float64[nf]  c_j^(i)
  p         perturbation probability

Nothing here computes anything the method computes; the dataclass only
carries arrays.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np


@dataclass
class PbnModel:
    n: int
    fn_off: np.ndarray
    par_off: np.ndarray
    parents: np.ndarray
    tbl_off: np.ndarray
    tables: np.ndarray
    sel_prob: np.ndarray
    p: float
    name: str = ""

    @property
    def nf(self) -> int:
        return int(self.fn_off[-1])

    def ell(self, i: int) -> int:
        return int(self.fn_off[i + 1] - self.fn_off[i])

    def theta(self, f: int) -> int:
        return int(self.par_off[f + 1] - self.par_off[f])

    def fn_parents(self, f: int) -> list[int]:
        return [int(x) for x in self.parents[self.par_off[f]:self.par_off[f + 1]]]

    def fn_table_bit(self, f: int, idx: int) -> int:
        w = int(self.tables[self.tbl_off[f] + (idx >> 5)])
        return (w >> (idx & 31)) & 1


@dataclass
class Predicate:
    """Property = conjunction of (node, value) pairs."""
    nodes: np.ndarray  # uint16[k]
    values: np.ndarray  # uint8[k]

    @property
    def k(self) -> int:
        return int(len(self.nodes))


@dataclass
class RunConfig:
    key: str
    n: int
    ell: tuple[int, int]
    theta: tuple[int, int]
    p: float
    table_bias: str          # "half" (Bernoulli(0.5)) or "uniform_q" (q ~ U(0.2,0.8) per function)
    model_seed: int
    sim_seed: int
    chains: int
    burn_in: int
    steps: int
    batch: int
    pred_nodes: tuple[int, ...]
    pred_values: tuple[int, ...]
    extra: dict = field(default_factory=dict)


# BASELINE.json configs; run protocol per SURVEY.md §8(d) table.
CONFIGS: dict[str, RunConfig] = {
    "C1": RunConfig("C1", 10, (2, 2), (1, 3), 0.01, "half", 1, 1,
                    chains=4, burn_in=1000, steps=10_000, batch=100,
                    pred_nodes=(0, 1), pred_values=(1, 1)),
    "C2": RunConfig("C2", 100, (1, 3), (1, 5), 0.001, "half", 2, 2,
                    chains=1024, burn_in=1000, steps=1000, batch=100,
                    pred_nodes=(0, 1, 2), pred_values=(1, 1, 1),
                    extra={"psi0": 1000, "rhat_threshold": 1.1, "r": 0.01,
                           "s": 0.95, "eps": 1e-10}),
    "C3": RunConfig("C3", 1000, (1, 3), (1, 5), 1e-4, "uniform_q", 3, 3,
                    chains=4096, burn_in=50_000, steps=50_000, batch=500,
                    pred_nodes=(0, 1, 2, 3, 4), pred_values=(1, 0, 1, 0, 1),
                    extra={"h_star": 1e-3, "alpha_conf": 0.05}),
    "C4": RunConfig("C4", 2000, (1, 4), (1, 6), 1e-4, "half", 4, 4,
                    chains=16384, burn_in=50_000, steps=50_000, batch=500,
                    pred_nodes=(0, 1, 2, 3, 4), pred_values=(1, 0, 1, 0, 1)),
    "C5": RunConfig("C5", 5000, (1, 4), (1, 8), 5e-5, "half", 5, 5,
                    chains=16384, burn_in=0, steps=10_000, batch=100,
                    pred_nodes=(0, 1, 2, 3, 4), pred_values=(1, 0, 1, 0, 1),
                    extra={"chain_sweep": (1, 64, 1024, 16384, 65536)}),
    # NEXT-3: the paper's DENSE class, density D = 150-300
    # (P:605-609); ell ~ U{8..24}, theta ~ U{8..12}: D ~ 16 x 10 = 160.
    # Not a BASELINE.json config (BASELINE's C1-C5 are all sparse).
    "C6": RunConfig("C6", 1000, (8, 24), (8, 12), 1e-4, "half", 6, 6,
                    chains=16384, burn_in=5_000, steps=5_000, batch=100,
                    pred_nodes=(0, 1, 2, 3, 4), pred_values=(1, 0, 1, 0, 1),
                    extra={"density_class": "dense"}),
}


def _pack_table(bits: np.ndarray) -> np.ndarray:
    """Pack 0/1 entries (index order) into uint32 words, LSB first: entry
    idx is bit (idx & 31) of word idx >> 5."""
    bits = np.asarray(bits, dtype=np.uint8)
    nw = (len(bits) + 31) // 32
    padded = np.zeros(nw * 32, dtype=np.uint8)
    padded[:len(bits)] = bits
    return np.packbits(padded, bitorder="little").view("<u4").astype(np.uint32)


def model_from_lists(n: int, p: float, nodes: list[list[tuple[list[int], list[int], float]]],
                     name: str = "") -> PbnModel:
    """Build a model from per-node lists of (parents, table_bits, prob).

    table_bits[idx] is f(x) for index idx formed with parents[0] as MSB.
    """
    assert len(nodes) == n
    fn_off = [0]
    par_off = [0]
    tbl_off = [0]
    parents: list[int] = []
    tables: list[np.ndarray] = []
    probs: list[float] = []
    for fns in nodes:
        for (par, bits, prob) in fns:
            assert len(bits) == (1 << len(par))
            parents.extend(par)
            par_off.append(len(parents))
            w = _pack_table(np.asarray(bits, dtype=np.uint8))
            tables.append(w)
            tbl_off.append(tbl_off[-1] + len(w))
            probs.append(prob)
        fn_off.append(len(probs))
    return PbnModel(
        n=n,
        fn_off=np.asarray(fn_off, dtype=np.int32),
        par_off=np.asarray(par_off, dtype=np.int32),
        parents=np.asarray(parents, dtype=np.uint16),
        tbl_off=np.asarray(tbl_off, dtype=np.int32),
        tables=(np.concatenate(tables) if tables else np.zeros(0, np.uint32)).astype(np.uint32),
        sel_prob=np.asarray(probs, dtype=np.float64),
        p=float(p),
        name=name,
    )


def random_pbn(n: int, f_min: int, f_max: int, par_min: int, par_max: int, p: float,
               seed: int, table_bias: str = "half", name: str = "") -> PbnModel:
    """Random PBN with the five ASSA-PBN generator parameters.

    Per node ell ~ U{f_min..f_max}; per function theta ~ U{par_min..par_max},
    parents uniform without replacement from all n nodes, Dirichlet(1^ell)
    selection probabilities, truth-table bits i.i.d. Bernoulli(0.5)
    ("half") or Bernoulli(q), q ~ U(0.2, 0.8) per function ("uniform_q").
    """
    if not (1 <= f_min <= f_max):
        raise ValueError("need 1 <= f_min <= f_max")
    if not (0 <= par_min <= par_max <= n):
        raise ValueError("need 0 <= par_min <= par_max <= n")
    rng = np.random.default_rng(seed)
    fn_off = [0]
    par_off = [0]
    tbl_off = [0]
    parents: list[np.ndarray] = []
    tables: list[np.ndarray] = []
    probs: list[np.ndarray] = []
    npar = 0
    for _ in range(n):
        ell = int(rng.integers(f_min, f_max + 1))
        c = rng.dirichlet(np.ones(ell)) if ell > 1 else np.ones(1)
        probs.append(np.asarray(c, dtype=np.float64))
        for _j in range(ell):
            theta = int(rng.integers(par_min, par_max + 1))
            par = rng.choice(n, size=theta, replace=False).astype(np.uint16)
            parents.append(par)
            npar += theta
            par_off.append(npar)
            q = 0.5 if table_bias == "half" else float(rng.uniform(0.2, 0.8))
            bits = (rng.random(1 << theta) < q).astype(np.uint8)
            w = _pack_table(bits)
            tables.append(w)
            tbl_off.append(tbl_off[-1] + len(w))
        fn_off.append(fn_off[-1] + ell)
    return PbnModel(
        n=n,
        fn_off=np.asarray(fn_off, dtype=np.int32),
        par_off=np.asarray(par_off, dtype=np.int32),
        parents=(np.concatenate(parents) if parents else np.zeros(0)).astype(np.uint16),
        tbl_off=np.asarray(tbl_off, dtype=np.int32),
        tables=np.concatenate(tables).astype(np.uint32),
        sel_prob=np.concatenate(probs).astype(np.float64),
        p=float(p),
        name=name,
    )


def config_model(key: str) -> PbnModel:
    c = CONFIGS[key]
    return random_pbn(c.n, c.ell[0], c.ell[1], c.theta[0], c.theta[1], c.p,
                      seed=c.model_seed, table_bias=c.table_bias, name=key)


def config_predicate(key: str) -> Predicate:
    c = CONFIGS[key]
    return Predicate(np.asarray(c.pred_nodes, dtype=np.uint16),
                     np.asarray(c.pred_values, dtype=np.uint8))

