"""Time pbn_simulate on C5 for forced cluster sizes (few-chain regime study)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1508_07828_b200 as pbn
from workloads import config_model, config_predicate
torch.cuda.set_device(0)
key = sys.argv[1] if len(sys.argv) > 1 else "C5"
model, pred = config_model(key), config_predicate(key)
pm = pbn.pbn_load(model)
steps = 2000
chain_list = [int(c) for c in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 64, 1024]
Ks = [int(c) for c in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 2, 4, 8, 16]
for chains in chain_list:
    for K in Ks:
        if K > (model.n + 3) // 4:
            continue
        out = pbn.alloc_outputs(pm, chains, steps, batch=100, emit_bits=True)
        def run():
            pbn.pbn_simulate(pm, out, n_chains=chains, steps=steps, batch=100, seed=5, pred=pred, init=True,
                             emit_bits=True, cluster_size=K)
        try:
            run(); torch.cuda.synchronize()
        except Exception as e:
            print(chains, K, "n/a", str(e)[:60]); continue
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run(); b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        print(key, chains, K, f"{ms:.2f} ms", f"{chains * steps * model.n / ms / 1e-3:.3g} node-updates/s", flush=True)
