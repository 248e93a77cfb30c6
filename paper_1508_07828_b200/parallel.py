"""Chain-level data parallelism across GPUs.

Chains are independent and every random word is keyed by the GLOBAL chain
id (reading Q2), so any partition of the chain range over ranks gives the
per-chain results of a single-GPU run bit for bit.  The only exchange the
method has is the pooled counters the host statistics consume (Alg 3 lines
6-9; the alpha/beta counts of Alg 4): six exact u64 sums,
reduced with one all-reduce.  Timing across ranks is the max.

Host logic only (torch.distributed; NCCL on the B200 box, gloo in the CPU
tests); no arithmetic of the method lives here.
"""
from __future__ import annotations

import numpy as np


def shard(n_chains_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block of global chain ids for `rank`: (chain_base, count).

    Blocks differ in size by at most one and cover 0..n_chains_total-1 in
    rank order."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("need world >= 1 and 0 <= rank < world")
    if n_chains_total < 0:
        raise ValueError("n_chains_total must be >= 0")
    q, r = divmod(n_chains_total, world)
    base = rank * q + min(rank, r)
    return base, q + (1 if rank < r else 0)


def allreduce_totals(totals, group=None) -> np.ndarray:
    """Sum the six u64 totals (S1, S2, n01, n10, n0from, n1from) over ranks.

    `totals` is a host array or a tensor of 6 non-negative integers < 2^63
    (u64 counts of one GPU's chains); returns the pooled u64 array.  The
    reduction runs on the device of the process group's backend (CUDA for
    NCCL, CPU for gloo)."""
    import torch
    import torch.distributed as dist

    t = totals if isinstance(totals, torch.Tensor) else torch.as_tensor(np.asarray(totals, dtype=np.uint64).view(np.int64))
    t = t.view(torch.int64).clone()
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    else:
        t = t.cpu()
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy().view(np.uint64)


def max_over_ranks(x: float, group=None) -> float:
    """Max of a per-rank float (device-timed milliseconds) over the group."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], dtype=torch.float64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.cpu()[0])


def run_sharded(model, *, omega: int, psi0: int, rhat_threshold: float = 1.1, r: float = 0.01,
                s: float = 0.95, eps: float = 1e-10, seed: int = 0, pred=None, max_steps: int = 1 << 26,
                method: int = 0, h_star: float = 1e-3, alpha_conf: float = 0.05, group=None, stream=None):
    """Algorithm 3 + Algorithm 4 (method 0) or 5 (method 1, Skart) over
    `omega` chains sharded across the ranks of `group` (one GPU each): this
    rank simulates its contiguous block of global chain ids; pooled numbers
    (six u64 counts per decision, or Skart's per-chain batch sums gathered
    chain-major) are summed with one all-reduce (pbn_run_sharded,
    include/pbnsim.h).  Every rank returns the same (status, pbn_run_result,
    err) as a single-GPU pbn_run over all chains.  Needs omega >= world (every
    rank simulates at least one chain)."""
    import ctypes as C
    import torch
    import torch.distributed as dist
    from . import _lib as L
    from .api import _pred, _stream_handle

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if omega < world:
        raise ValueError(f"omega={omega} chains cannot be sharded over {world} ranks (each needs >= 1)")
    base, count = shard(omega, world, rank)
    nccl = dist.get_backend(group) == "nccl"
    state = {"error": None}

    def _allreduce(values, n, ctx):
        try:
            v = np.ctypeslib.as_array(values, shape=(n,)).view(np.int64)
            t = torch.from_numpy(v.copy())
            if nccl:
                t = t.cuda()
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
            v[:] = t.cpu().numpy()
            return 0
        except Exception as e:  # reported through the status, never raised across C
            state["error"] = e
            return 1

    cb = L.ALLREDUCE_FN(_allreduce)
    cp, _keep = _pred(pred)
    a = L.pbn_run_args(method=method, omega=omega, psi0=psi0, rhat_threshold=rhat_threshold, r=r, s=s, eps=eps,
                       h_star=h_star, alpha_conf=alpha_conf, seed=seed, pred=cp, max_steps=max_steps)
    res = L.pbn_run_result()
    err = C.create_string_buffer(512)
    st = L.lib().pbn_run_sharded(model.handle, C.byref(a), base, count, C.cast(cb, C.c_void_p), None,
                                 C.byref(res), _stream_handle(stream), err, 512)
    msg = err.value.decode(errors="replace")
    if state["error"] is not None:
        msg = f"all-reduce failed: {state['error']}"
    return st, res, msg
