# parity + bench + ncu capture of one short K1 launch (C4, 2000 recorded steps)
TAG=${1:-iter}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
grep -o '"value": [0-9.e+]*, "unit": "node-updates/s", "n_gpus"' gpurun_out/bench_$TAG.log | head -1
grep -o '"frac": [0-9.e+-]*' gpurun_out/bench_$TAG.log
bash scripts/profile.sh $TAG --burn-in 0 --window 2000 > /dev/null 2>&1; echo "profile rc=$?"
