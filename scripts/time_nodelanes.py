"""Lanes-over-nodes (K1n) grid: node-updates/s for every cluster size K and
chains per cluster G, next to the auto choice and the chain-lanes kernels."""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1508_07828_b200 as pbn  # noqa: E402
from workloads import config_model, config_predicate  # noqa: E402

keys = sys.argv[1].split(",")
chain_list = [int(x) for x in sys.argv[2].split(",")]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
for key in keys:
    model, pred = config_model(key), config_predicate(key)
    pm = pbn.pbn_load(model)
    for chains in chain_list:
        out = pbn.alloc_outputs(pm, chains, steps, batch=100, emit_bits=True)
        variants = [("auto", 0, 0, 0), ("chain-lanes", 1, 0, 0), ("node-lanes auto", 2, 0, 0)]
        variants += [(f"node-lanes K={K} G={G}", 2, K, G) for K in (1, 2, 4, 8, 16) for G in (1, 2, 4, 8, 16, 32)
                     if G <= max(1, chains)]
        for name, layout, K, G in variants:
            def run():
                pbn.pbn_simulate(pm, out, n_chains=chains, steps=steps, batch=100, seed=1, pred=pred, init=True,
                                 emit_bits=True, layout=layout, cluster_size=K, chains_per_cluster=G)
            try:
                run()
                torch.cuda.synchronize()
            except Exception:
                continue
            ms = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                run()
                b.record()
                torch.cuda.synchronize()
                ms.append(a.elapsed_time(b))
            t = statistics.median(ms) / 1e3
            print(json.dumps({"config": key, "chains": chains, "variant": name,
                              "node_updates_per_s": chains * steps * model.n / t, "us_per_step": t / steps * 1e6}),
                  flush=True)
    pm.close()
