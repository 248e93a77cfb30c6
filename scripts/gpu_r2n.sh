# global-image K1: parity subset + C5 16384/65536 and C6 timings
TAG=${1:-r2n}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf -k "global_image or large_configs or dense or maximum or geometric_mode_C4" > gpurun_out/pytest_gi_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gi_$TAG.log
for c in 16384 65536; do
  timeout 600 python bench.py --config C5 --chains $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C5_${c}_$TAG.log 2>&1; echo "C5 $c rc=$?"
  tail -1 gpurun_out/bench_C5_${c}_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'].get('n_chains', ''), d['value'], d['roofline']['frac'], d.get('ms_per_step'))"
done
timeout 600 python bench.py --config C6 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C6_$TAG.log 2>&1; echo "C6 rc=$?"
tail -1 gpurun_out/bench_C6_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C6', d['value'], d['roofline']['frac'])"
