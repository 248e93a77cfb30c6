# parity + bench + short-run profile of the traj kernel
TAG=${1:-iter}
timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
true <<'PY'
import json,sys
l=[x for x in open("gpurun_out/bench_%s.log" % sys.argv[1] if len(sys.argv)>1 else "gpurun_out/bench_iter.log") if x.startswith('{')]
PY
grep -o '"value": [0-9.e+]*, "unit": "node-updates/s", "n_gpus"' gpurun_out/bench_$TAG.log | head -1
grep -o '"frac": [0-9.e+-]*' gpurun_out/bench_$TAG.log
bash scripts/profile.sh $TAG --burn-in 0 --window 400 > /dev/null 2>&1; echo "profile rc=$?"
