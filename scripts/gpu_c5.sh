# full GPU tests, then the C5 chain-count sweep (BASELINE config 5), 10^4 steps per chain
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_c5.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_c5.log
timeout 1500 python bench.py --sweep --steps 3 --warmup 3 > gpurun_out/sweep_c5.log 2>&1; echo "sweep rc=$?"
grep sweep gpurun_out/sweep_c5.log | cut -c1-300
