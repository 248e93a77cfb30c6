"""Pins for the oracle's Philox4x32-10 and its stream definition.

Pin: cuRAND's header implementation `curand_Philox4x32_10`
(/usr/local/cuda/include/curand_philox4x32_x.h), compiled for the host by
nvcc -- an independent implementation of the published generator
(Salmon et al., SC'11).  Stream layout pins follow DESIGN.md reading Q2.
"""
import ctypes as C
import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle import sim

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def curand_host(tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    out = str(tmp_path_factory.mktemp("pin") / "curand_philox_host.so")
    subprocess.check_call([nvcc, "-shared", "-Xcompiler", "-fPIC", "-Wno-deprecated-gpu-targets",
                           "-o", out, os.path.join(HERE, "pins", "curand_philox_host.cu")])
    L = C.CDLL(out)
    L.curand_philox_host.argtypes = [np.ctypeslib.ndpointer(np.uint32)] * 3 + [C.c_int]
    return L


def test_philox_matches_curand(curand_host):
    rng = np.random.default_rng(1234)
    count = 2000
    ctr = rng.integers(0, 2**32, size=(count, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2**32, size=(count, 2), dtype=np.uint64).astype(np.uint32)
    # include edge counters / keys
    ctr[0] = 0
    key[0] = 0
    ctr[1] = 0xFFFFFFFF
    key[1] = 0xFFFFFFFF
    ref = np.zeros((count, 4), np.uint32)
    curand_host.curand_philox_host(np.ascontiguousarray(ctr), np.ascontiguousarray(key), ref, count)
    got = np.stack([sim.philox4x32_10(ctr[i], key[i]) for i in range(count)])
    assert np.array_equal(got, ref)


def test_stream_layout(curand_host):
    """u(chain,t,i) = philox((i//4, chain, t lo, t hi), (seed lo, seed hi))[i%4]."""
    seed = 0x1234_5678_9ABC_DEF0
    for chain, t, i in [(0, 0, 0), (5, 1, 3), (7, 2**32 + 5, 9), (2**31, 123456, 4001)]:
        ctr = np.array([i // 4, chain, t & 0xFFFFFFFF, t >> 32], np.uint32)
        key = np.array([seed & 0xFFFFFFFF, seed >> 32], np.uint32)
        ref = np.zeros(4, np.uint32)
        curand_host.curand_philox_host(ctr, key, ref, 1)
        assert sim.word(seed, chain, t, i) == int(ref[i % 4])


def test_words_look_uniform():
    """Coarse sanity: 4096 words of one stream spread over 16 bins (chi^2)."""
    w = np.array([sim.word(7, 3, t, i) for t in range(1, 65) for i in range(64)], np.uint64)
    hist = np.bincount((w >> 28).astype(np.int64), minlength=16)
    exp = len(w) / 16
    chi2 = float(np.sum((hist - exp) ** 2 / exp))
    assert chi2 < 50.0  # 15 dof; p ~ 1e-5
