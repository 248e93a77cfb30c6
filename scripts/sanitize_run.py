"""Small launches of every kernel path for compute-sanitizer (racecheck / memcheck / synccheck):
K1 VECTOR and PER_NODE (single CTA per group, persistent chunks), K1c clusters, K2 recount."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1508_07828_b200 as pbn
from workloads import config_model, config_predicate

torch.cuda.set_device(0)
for key in ("C1", "C2"):
    model, pred = config_model(key), config_predicate(key)
    for per_node in (False, True):
        pm = pbn.pbn_load(model, per_node=per_node)
        for cl, sched in ((1, 1), (1, 2), (2, 0), (4, 0)):
            if cl > 1 and (model.n + 3) // 4 < cl:
                continue
            out = pbn.alloc_outputs(pm, 70, 120, batch=16, emit_bits=True, n_props=2)
            pbn.pbn_simulate(pm, out, n_chains=70, steps=120, burn_in=30, batch=16, seed=3, init=True,
                             emit_bits=True, props=[pred, pred], cluster_size=cl, schedule=sched,
                             chunk_steps=17 if sched == 2 else 0)
            torch.cuda.synchronize()
        c1 = torch.empty(70, dtype=torch.int32, device="cuda")
        pbn.pbn_recount(out.bits[0], 70, out.bits.shape[2], 5, 100, 10, c1, None, None, None,
                        torch.empty((70, 10), dtype=torch.int32, device="cuda"), None)
        torch.cuda.synchronize()
        pm.close()
print("sanitize run done")
