TAG=${1:-r2m}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf -k "geometric or node_lanes" > gpurun_out/pytest_geo_$TAG.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_geo_$TAG.log
cat > /tmp/geo_time.py <<'PY'
import sys, json, statistics, torch
sys.path.insert(0, ".")
import paper_1508_07828_b200 as pbn
from workloads import config_model, config_predicate
for key in ["C5", "C4"]:
    model, pred = config_model(key), config_predicate(key)
    for geo in (False, True):
        pm = pbn.pbn_load(model, geometric=geo)
        for chains in (1, 64):
            out = pbn.alloc_outputs(pm, chains, 2000, batch=100, emit_bits=True)
            run = lambda: pbn.pbn_simulate(pm, out, n_chains=chains, steps=2000, batch=100, seed=1, pred=pred, init=True, emit_bits=True)
            run(); torch.cuda.synchronize()
            ms = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); run(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
            t = statistics.median(ms) / 1e3
            print(json.dumps({"config": key, "geometric": geo, "chains": chains, "node_updates_per_s": chains * 2000 * model.n / t}))
        pm.close()
PY
timeout 600 python /tmp/geo_time.py
