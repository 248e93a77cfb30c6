TAG=${1:-r2j}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf -k "geometric" > gpurun_out/pytest_geo_$TAG.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/pytest_geo_$TAG.log
timeout 900 python bench.py --geometric --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_geo_$TAG.log 2>&1; echo "bench geo rc=$?"; tail -1 gpurun_out/bench_geo_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['bound'], d['roofline']['frac'], d['config']['semantics'])"
