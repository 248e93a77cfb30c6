# ncu --set full of K1b-global (C5 16384 chains) and K1bc (C5 1024 chains, K = 4), short windows
TAG=${1:-r3y}
mkdir -p gpurun_out
CMD="python bench.py --config C5 --chains 16384 --burn-in 0 --window 500 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain_${TAG}g.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:bitslice_kernel -s 3 -c 1 -o gpurun_out/prof_${TAG}g $CMD > gpurun_out/ncu_${TAG}g.log 2>&1; echo "global rc=$?"
CMD="python bench.py --config C5 --chains 1024 --burn-in 0 --window 2000 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain_${TAG}c.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:bitslice_kernel -s 3 -c 1 -o gpurun_out/prof_${TAG}c $CMD > gpurun_out/ncu_${TAG}c.log 2>&1; echo "cluster rc=$?"
