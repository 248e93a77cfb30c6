# generalized K1b (binary planes, classes to 8, global image): its tests, C5 parity, C4/C3/C5 numbers
TAG=${1:-r3p}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bitslice_gpu.py -x -q -rf > gpurun_out/pytest_bs_$TAG.log 2>&1; echo "pytest bs rc=$?"; tail -3 gpurun_out/pytest_bs_$TAG.log
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -rf -k "large_configs" > gpurun_out/pytest_large_$TAG.log 2>&1; echo "pytest large rc=$?"; tail -3 gpurun_out/pytest_large_$TAG.log
CONFIGS="C4 C3" bash scripts/gpu_bsab2.sh $TAG default:28
timeout 900 python bench.py --sweep --steps 3 --warmup 3 > gpurun_out/sweep_$TAG.jsonl 2>&1; echo "sweep rc=$?"; cut -c1-200 gpurun_out/sweep_$TAG.jsonl
PBN_NO_BITSLICE=1 timeout 900 python bench.py --sweep --steps 3 --warmup 3 > gpurun_out/sweep_nobs_$TAG.jsonl 2>&1; echo "sweep (no K1b) rc=$?"; cut -c1-200 gpurun_out/sweep_nobs_$TAG.jsonl
