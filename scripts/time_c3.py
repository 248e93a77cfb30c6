import os, sys
sys.path.insert(0, '/root/repo')
import torch
import paper_1508_07828_b200 as pbn
from workloads import config_model, config_predicate
torch.cuda.set_device(0)
model, pred = config_model("C3"), config_predicate("C3")
pm = pbn.pbn_load(model)
steps = 5000
for chains in (2048, 4096, 8192):
    for K in (0, 1, 2, 4):
        out = pbn.alloc_outputs(pm, chains, steps, batch=500, emit_bits=True)
        run = lambda: pbn.pbn_simulate(pm, out, n_chains=chains, steps=steps, batch=500, seed=5, pred=pred, init=True, emit_bits=True, cluster_size=K)
        try:
            run(); torch.cuda.synchronize()
        except Exception as e:
            print(chains, K, 'n/a'); continue
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run(); b.record(); torch.cuda.synchronize()
        print(chains, K, f"{chains*steps*model.n/a.elapsed_time(b)/1e-3:.3g}", flush=True)
