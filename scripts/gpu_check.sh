nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q --durations=10 > gpurun_out/pytest_gpu1.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu1.log
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench1.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/bench1.log
