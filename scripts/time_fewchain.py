"""Few-chain regime: node-updates/s of the chain-lanes kernels (auto: K1c)
vs lanes over nodes (K1n) at each cluster size, C2-C5, 1 / 64 / 256 chains."""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1508_07828_b200 as pbn  # noqa: E402
from workloads import CONFIGS, config_model, config_predicate  # noqa: E402

keys = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C5", "C4", "C3", "C2"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
for key in keys:
    model, pred = config_model(key), config_predicate(key)
    pm = pbn.pbn_load(model)
    for chains in (1, 64, 256):
        out = pbn.alloc_outputs(pm, chains, steps, batch=100, emit_bits=True)
        variants = [("auto", 0, 0), ("chain-lanes", 1, 0)] + [(f"node-lanes K={K}", 2, K) for K in (1, 2, 4, 8, 16)]
        for name, layout, K in variants:
            def run():
                pbn.pbn_simulate(pm, out, n_chains=chains, steps=steps, batch=100, seed=1, pred=pred, init=True,
                                 emit_bits=True, layout=layout, cluster_size=K)
            try:
                run()
                torch.cuda.synchronize()
            except Exception as e:
                print(json.dumps({"config": key, "chains": chains, "variant": name, "error": str(e)[:80]}))
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
