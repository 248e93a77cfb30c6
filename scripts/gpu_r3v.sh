# K1bc first light: tests, C5 1024 / C2 / C3 timing vs K1c / K1b
TAG=${1:-r3v}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bitslice_gpu.py -x -q -rf -k "cluster" > gpurun_out/pytest_bsc_$TAG.log 2>&1; echo "pytest cluster rc=$?"; tail -15 gpurun_out/pytest_bsc_$TAG.log
for K in 2 4 8; do
  timeout 300 python bench.py --config C5 --chains 1024 --layout 3 --cluster $K --burn-in 0 --window 10000 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bsc_${TAG}_C5_$K.log 2>&1; echo "C5 1024 K1bc K=$K rc=$? $(grep -o '"value": [0-9.e+]*' gpurun_out/bsc_${TAG}_C5_$K.log | head -1)"
done
timeout 300 python bench.py --config C5 --chains 1024 --burn-in 0 --window 10000 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bsc_${TAG}_C5_auto.log 2>&1; echo "C5 1024 auto rc=$? $(grep -o '"value": [0-9.e+]*' gpurun_out/bsc_${TAG}_C5_auto.log | head -1)"
for K in 2 4; do
  timeout 300 python bench.py --config C2 --chains 1024 --layout 3 --cluster $K --burn-in 0 --window 20000 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bsc_${TAG}_C2_$K.log 2>&1; echo "C2 1024 K1bc K=$K rc=$? $(grep -o '"value": [0-9.e+]*' gpurun_out/bsc_${TAG}_C2_$K.log | head -1)"
done
timeout 300 python bench.py --config C2 --chains 1024 --burn-in 0 --window 20000 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bsc_${TAG}_C2_auto.log 2>&1; echo "C2 1024 auto rc=$? $(grep -o '"value": [0-9.e+]*' gpurun_out/bsc_${TAG}_C2_auto.log | head -1)"
