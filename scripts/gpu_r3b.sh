# K1b first light: its parity tests, then C4 / C3 bench lines through layout 3
TAG=${1:-r3b}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bitslice_gpu.py -x -q -rf --durations=5 > gpurun_out/pytest_bs_$TAG.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_bs_$TAG.log
timeout 600 python bench.py --layout 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_bs_C4_$TAG.log 2>&1; echo "bench C4 rc=$?"; tail -1 gpurun_out/bench_bs_C4_$TAG.log | cut -c1-400
timeout 600 python bench.py --layout 3 --config C3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_bs_C3_$TAG.log 2>&1; echo "bench C3 rc=$?"; tail -1 gpurun_out/bench_bs_C3_$TAG.log | cut -c1-400
