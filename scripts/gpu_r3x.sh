TAG=${1:-r3x}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=5 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --sweep --steps 3 --warmup 3 > gpurun_out/sweep_$TAG.jsonl 2>&1; echo "sweep rc=$?"; cut -c1-160 gpurun_out/sweep_$TAG.jsonl
timeout 1200 python bench.py --protocol C2,C3 > gpurun_out/protocol_$TAG.jsonl 2>&1; echo "protocol rc=$?"
