TAG=${1:-r2g}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -16 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --sweep --steps 3 --warmup 3 > gpurun_out/sweep_$TAG.jsonl 2>&1; echo "sweep rc=$?"; cut -c1-300 gpurun_out/sweep_$TAG.jsonl
timeout 900 python scripts/time_nodelanes.py C5,C4,C3,C2 1,64,256,1024 1000 > gpurun_out/nodelanes_$TAG.jsonl 2>&1; echo "grid rc=$?"
grep '"auto"\|chain-lanes\|node-lanes auto' gpurun_out/nodelanes_$TAG.jsonl | cut -c1-160
