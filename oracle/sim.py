"""ctypes marshalling for the plain C oracle (oracle/pbn_oracle.c).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _build

_lib = None
_lock = threading.Lock()

_p = np.ctypeslib.ndpointer


def lib():
    global _lib
    with _lock:
        if _lib is None:
            path = _build.build()
            L = C.CDLL(path)
            L.oracle_philox4x32_10.argtypes = [_p(np.uint32, flags="C"), _p(np.uint32, flags="C"),
                                               _p(np.uint32, flags="C")]
            L.oracle_philox4x32_10.restype = None
            L.oracle_word.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32]
            L.oracle_word.restype = C.c_uint32
            L.oracle_perturbation_threshold.argtypes = [C.c_double]
            L.oracle_perturbation_threshold.restype = C.c_uint32
            L.oracle_selection_thresholds.argtypes = [C.c_int32, _p(np.int32, flags="C"),
                                                      _p(np.float64, flags="C"), C.c_double,
                                                      _p(np.uint64, flags="C")]
            L.oracle_selection_thresholds.restype = None
            model_args = [C.c_int32, _p(np.int32, flags="C"), _p(np.int32, flags="C"),
                          _p(np.uint16, flags="C"), _p(np.int32, flags="C"),
                          _p(np.uint32, flags="C"), _p(np.float64, flags="C"), C.c_double,
                          C.c_int32]
            L.oracle_step.argtypes = model_args + [_p(np.uint8, flags="C"),
                                                   _p(np.uint32, flags="C"),
                                                   _p(np.uint8, flags="C")]
            L.oracle_step.restype = C.c_int
            L.oracle_simulate.argtypes = model_args + [
                C.c_uint64, _p(np.uint32, flags="C"), C.c_int64, C.c_int64, C.c_int64,
                C.c_int64, C.c_int32, C.c_int32, _p(np.uint16, flags="C"),
                _p(np.uint8, flags="C"), _p(np.uint8, flags="C"), _p(np.uint8, flags="C")]
            L.oracle_simulate.restype = C.c_int
            L.oracle_geometric_table.argtypes = [C.c_int32, C.c_double, _p(np.uint32, flags="C")]
            L.oracle_geometric_table.restype = None
            L.oracle_skip_word.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32]
            L.oracle_skip_word.restype = C.c_uint32
            L.oracle_skip.argtypes = [_p(np.uint32, flags="C"), C.c_int32, C.c_uint32]
            L.oracle_skip.restype = C.c_int32
            _lib = L
    return _lib


def _model_args(model, per_node: bool):
    parents = np.ascontiguousarray(model.parents, dtype=np.uint16)
    if parents.size == 0:
        parents = np.zeros(1, np.uint16)
    return (int(model.n), np.ascontiguousarray(model.fn_off, np.int32),
            np.ascontiguousarray(model.par_off, np.int32), parents,
            np.ascontiguousarray(model.tbl_off, np.int32),
            np.ascontiguousarray(model.tables, np.uint32),
            np.ascontiguousarray(model.sel_prob, np.float64), float(model.p), int(per_node))


def philox4x32_10(ctr, key) -> np.ndarray:
    out = np.zeros(4, np.uint32)
    lib().oracle_philox4x32_10(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
    return out


def word(seed: int, chain: int, t: int, i: int) -> int:
    return int(lib().oracle_word(seed, chain, t, i))


def perturbation_threshold(p: float) -> int:
    return int(lib().oracle_perturbation_threshold(p))


def selection_thresholds(model) -> np.ndarray:
    D = np.zeros(max(model.nf, 1), np.uint64)
    lib().oracle_selection_thresholds(int(model.n), np.ascontiguousarray(model.fn_off, np.int32),
                                      np.ascontiguousarray(model.sel_prob, np.float64),
                                      float(model.p), D)
    return D[:model.nf]


def step(model, s, u, per_node: bool = False) -> np.ndarray:
    s = np.ascontiguousarray(s, np.uint8)
    u = np.ascontiguousarray(u, np.uint32)
    out = np.zeros(model.n, np.uint8)
    rc = lib().oracle_step(*_model_args(model, per_node), s, u, out)
    assert rc == 0
    return out


def geometric_table(model) -> np.ndarray:
    Cg = np.zeros(max(int(model.n), 1), np.uint32)
    lib().oracle_geometric_table(int(model.n), float(model.p), Cg)
    return Cg[:model.n]


def skip_word(seed: int, chain: int, t: int, m: int) -> int:
    return int(lib().oracle_skip_word(seed, chain, t, m))


def skip(Cg: np.ndarray, v: int) -> int:
    Cg = np.ascontiguousarray(Cg, np.uint32)
    return int(lib().oracle_skip(Cg, len(Cg), int(v)))


def simulate(model, pred, seed: int, chain_ids, step0: int, burn_in: int, steps: int,
             init: bool = True, state=None, per_node: bool = False, threads: int = 1,
             geometric: bool = False):
    """Run the oracle trajectories.

    Returns (state [nchains x n] uint8 = s_{step0+burn_in+steps},
             I [nchains x steps] uint8 = indicator over the recorded window).
    geometric: VECTOR semantics with the geometric-skip perturbation stream
    (NEXT-2, reading Q18).
    With threads > 1 the chain list is split over a thread pool (the C call
    releases the GIL); results do not depend on the split.
    """
    chain_ids = np.ascontiguousarray(chain_ids, np.uint32)
    nch = len(chain_ids)
    n = int(model.n)
    if state is None:
        assert init, "need a state when init is False"
        st = np.zeros((nch, n), np.uint8)
    else:
        st = np.array(state, dtype=np.uint8, copy=True).reshape(nch, n)
    I = np.zeros((nch, max(steps, 0)), np.uint8)
    if geometric and per_node:
        raise ValueError("the geometric-skip stream is defined for VECTOR semantics (reading Q18)")
    margs = _model_args(model, 2 if geometric else per_node)
    pn = np.ascontiguousarray(pred.nodes, np.uint16) if pred.k else np.zeros(1, np.uint16)
    pv = np.ascontiguousarray(pred.values, np.uint8) if pred.k else np.zeros(1, np.uint8)

    def run(lo: int, hi: int):
        if hi <= lo:
            return
        sub_state = np.ascontiguousarray(st[lo:hi])
        sub_I = np.zeros((hi - lo, max(steps, 1)), np.uint8)
        rc = lib().oracle_simulate(*margs, int(seed), np.ascontiguousarray(chain_ids[lo:hi]),
                                   hi - lo, int(step0), int(burn_in), int(steps), int(init),
                                   int(pred.k), pn, pv, sub_state, sub_I)
        assert rc == 0, rc
        st[lo:hi] = sub_state
        if steps > 0:
            I[lo:hi] = sub_I[:, :steps]

    threads = max(1, min(int(threads), nch)) if nch else 1
    if threads == 1:
        run(0, nch)
    else:
        bounds = np.linspace(0, nch, threads + 1).astype(int)
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda a: run(*a), zip(bounds[:-1], bounds[1:])))
    return st, I


def host_cores() -> int:
    return len(os.sched_getaffinity(0))
