timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pytest_sw0.log 2>&1; echo "pytest default rc=$?"
PBN_STATS_WARPS=1 timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pytest_sw1.log 2>&1; echo "pytest statswarp rc=$?"; tail -1 gpurun_out/pytest_sw1.log
for i in 1 2; do
for V in 0 1; do echo -n "STATS_WARPS=$V "; PBN_STATS_WARPS=$V timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -o '"value": [0-9.e+]*' | head -1; done
done
