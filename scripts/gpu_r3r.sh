# K1b geometric mode: tests, the C4 geometric bench line
TAG=${1:-r3r}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bitslice_gpu.py -x -q -rf > gpurun_out/pytest_bs_$TAG.log 2>&1; echo "pytest bs rc=$?"; tail -3 gpurun_out/pytest_bs_$TAG.log
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -rf -k "geometric" > gpurun_out/pytest_geo_$TAG.log 2>&1; echo "pytest geo rc=$?"; tail -3 gpurun_out/pytest_geo_$TAG.log
timeout 900 python bench.py --geometric --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_geo_$TAG.log 2>&1; echo "geo rc=$?"; tail -1 gpurun_out/bench_geo_$TAG.log | cut -c1-200
