"""N > 1 host path on CPU: world_size-2 gloo processes shard the chains of one
run (paper_1508_07828_b200.parallel), compute their shard's per-chain window
statistics (here with the CPU oracle, standing in for each rank's GPU), and
all-reduce the six pooled u64 totals -- the only exchange of the method
(Alg 3 lines 6-9; Alg 4's alpha/beta counts).  The pooled
totals, and the R-hat / two-state values computed from them, must equal a
single-process run over all chains.
"""
import os
import socket
import tempfile

import numpy as np
import pytest

from paper_1508_07828_b200 import parallel


def test_shard_covers_range_in_rank_order():
    for total in [0, 1, 5, 37, 16384]:
        for world in [1, 2, 3, 8]:
            blocks = [parallel.shard(total, world, r) for r in range(world)]
            assert sum(c for _, c in blocks) == total
            nxt = 0
            for base, cnt in blocks:
                assert base == nxt
                nxt += cnt
            assert max(c for _, c in blocks) - min(c for _, c in blocks) <= 1
    with pytest.raises(ValueError):
        parallel.shard(10, 2, 2)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CHAINS, STEPS, BURN, SEED, BATCH = 37, 300, 50, 7, 25


def _rank_main(rank: int, world: int, port: int, outdir: str):
    import torch.distributed as dist
    from oracle import sim as osim
    from oracle import stats as ostats
    from workloads import config_model, config_predicate

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model, pred = config_model("C2"), config_predicate("C2")
    base, cnt = parallel.shard(CHAINS, world, rank)
    _, I = osim.simulate(model, pred, seed=SEED, chain_ids=np.arange(base, base + cnt), step0=0,
                         burn_in=BURN, steps=STEPS)
    ws = [ostats.window_stats(I[c], BATCH) for c in range(cnt)]
    local = ostats.totals(ws) if cnt else np.zeros(6, np.uint64)
    pooled = parallel.allreduce_totals(local)
    t = parallel.max_over_ranks(float(rank + 1))
    np.save(os.path.join(outdir, f"pooled_{rank}.npy"), pooled)
    np.save(os.path.join(outdir, f"max_{rank}.npy"), np.array([t]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_pooled_totals_equal_single_run():
    import torch.multiprocessing as mp
    from oracle import sim as osim
    from oracle import stats as ostats
    from workloads import config_model, config_predicate

    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank_main, args=(world, _free_port(), d), nprocs=world, join=True)
        pooled = [np.load(os.path.join(d, f"pooled_{r}.npy")) for r in range(world)]
        maxes = [float(np.load(os.path.join(d, f"max_{r}.npy"))[0]) for r in range(world)]
    model, pred = config_model("C2"), config_predicate("C2")
    _, I = osim.simulate(model, pred, seed=SEED, chain_ids=np.arange(CHAINS), step0=0, burn_in=BURN,
                         steps=STEPS)
    ws = [ostats.window_stats(I[c], BATCH) for c in range(CHAINS)]
    single = ostats.totals(ws)
    for p in pooled:
        assert np.array_equal(p, single)
    assert maxes == [2.0, 2.0]
    # the library's host R-hat from the pooled totals equals the oracle's
    # textbook two-pass R-hat over all chains (1e-9 relative, BJ)
    import paper_1508_07828_b200 as pbn
    c = np.array([w.c1 for w in ws], dtype=np.int64)
    ref = ostats.gelman_rubin_counts(c, STEPS)
    st, rhat, B, W, _ = pbn.pbn_gelman_rubin(int(pooled[0][0]), int(pooled[0][1]), CHAINS, STEPS)
    assert st == 0
    assert abs(rhat - ref.rhat) <= 1e-9 * abs(ref.rhat)
