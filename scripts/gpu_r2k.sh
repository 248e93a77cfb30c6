TAG=${1:-r2k}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x -k "node_lanes or C5" > gpurun_out/pytest_nl_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_nl_$TAG.log
timeout 1200 python scripts/time_nodelanes.py C5,C4,C3 1,64,256,1024 1000 > gpurun_out/nodelanes_$TAG.jsonl 2>&1; echo "grid rc=$?"
python - <<'PY'
import json
rows=[json.loads(l) for l in open("gpurun_out/nodelanes_r2k.jsonl") if l.startswith("{")]
from collections import defaultdict
best=defaultdict(lambda:(0,""))
for r in rows:
    k=(r["config"], r["chains"])
    if r["variant"].startswith("node-lanes K") and r["node_updates_per_s"]>best[k][0]: best[k]=(r["node_updates_per_s"], r["variant"])
for r in rows:
    if r["variant"] in ("auto","chain-lanes","node-lanes auto"): print(r["config"], r["chains"], r["variant"], "%.3g"%r["node_updates_per_s"])
for k,v in sorted(best.items()): print("BEST", k, "%.3g"%v[0], v[1])
PY
