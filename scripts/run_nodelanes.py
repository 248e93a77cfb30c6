"""One lanes-over-nodes launch for ncu: python scripts/run_nodelanes.py <config> <chains> <K> <steps>"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1508_07828_b200 as pbn  # noqa: E402
from workloads import config_model, config_predicate  # noqa: E402

key, chains, K, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
G = int(sys.argv[5]) if len(sys.argv) > 5 else 0
model, pred = config_model(key), config_predicate(key)
pm = pbn.pbn_load(model)
out = pbn.alloc_outputs(pm, chains, steps, batch=100, emit_bits=True)
for _ in range(2):
    pbn.pbn_simulate(pm, out, n_chains=chains, steps=steps, batch=100, seed=1, pred=pred, init=True, emit_bits=True,
                     layout=2, cluster_size=K, chains_per_cluster=G)
torch.cuda.synchronize()
print("ok")
