TAG=${1:-r2h}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf -k "dense or edge_models or maximum" > gpurun_out/pytest_dense_$TAG.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/pytest_dense_$TAG.log
timeout 900 python bench.py --config C6 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C6_$TAG.log 2>&1; echo "bench C6 rc=$?"; tail -1 gpurun_out/bench_C6_$TAG.log | cut -c1-2500
