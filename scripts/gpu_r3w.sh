# K1bc vs the auto kernels (K1n <= 256 chains, K1c 1024) on the sweep shapes
TAG=${1:-r3w}
mkdir -p gpurun_out
run() { # config chains window label args...
  CF=$1; CH=$2; WIN=$3; LB=$4; shift 4
  timeout 300 python bench.py --config $CF --chains $CH --burn-in 0 --window $WIN --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" > gpurun_out/sw_${TAG}_${CF}_${CH}_$LB.log 2>&1
  echo "$CF $CH $LB rc=$? $(grep -o '"value": [0-9.e+]*' gpurun_out/sw_${TAG}_${CF}_${CH}_$LB.log | head -1) $(grep -o '"kernel": "[^"]*"' gpurun_out/sw_${TAG}_${CF}_${CH}_$LB.log | tail -1)"
}
for CH in 64 256; do
  run C5 $CH 4000 auto
  for K in 8 16; do run C5 $CH 4000 bc$K --layout 3 --cluster $K; done
  run C4 $CH 4000 auto
  for K in 8 16; do run C4 $CH 4000 bc$K --layout 3 --cluster $K; done
done
run C4 1024 10000 auto
for K in 2 4 8; do run C4 1024 10000 bc$K --layout 3 --cluster $K; done
run C3 1024 10000 auto
for K in 2 4 8; do run C3 1024 10000 bc$K --layout 3 --cluster $K; done
run C3 2048 10000 auto
for K in 2 4; do run C3 2048 10000 bc$K --layout 3 --cluster $K; done
