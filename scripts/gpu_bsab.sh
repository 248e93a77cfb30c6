# K1b A/B: library variants x warps per group on C4 (20000 recorded steps) and C3
# usage: bash scripts/gpu_bsab.sh <tag> <variant.so> ...  ("default" = libpbnsim.so); WARPS="20 24 28"
TAG=$1; shift
mkdir -p gpurun_out
for V in "$@"; do
  if [ "$V" = default ]; then unset PBN_LIB_VARIANT; else export PBN_LIB_VARIANT=$V; fi
  for W in ${WARPS:-20 24 28}; do
    for CF in ${CONFIGS:-C4}; do
      timeout 300 python bench.py --config $CF --layout 3 --warps $W --burn-in 0 --window ${WINDOW:-20000} --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bsab_${TAG}_${V}_${W}_$CF.log 2>&1
      echo "$V warps=$W $CF rc=$? $(grep -o '"value": [0-9.e+]*' gpurun_out/bsab_${TAG}_${V}_${W}_$CF.log | head -1)"
    done
  done
done
