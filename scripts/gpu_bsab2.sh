# K1b thread-budget variants: <variant.so>:<warps> pairs on C4/C3 (20000 steps)
TAG=$1; shift
mkdir -p gpurun_out
for VW in "$@"; do
  V=${VW%%:*}; W=${VW##*:}
  if [ "$V" = default ]; then unset PBN_LIB_VARIANT; else export PBN_LIB_VARIANT=$V; fi
  for CF in ${CONFIGS:-C4}; do
    timeout 300 python bench.py --config $CF --warps $W --burn-in 0 --window ${WINDOW:-20000} --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bsab_${TAG}_${V}_${W}_$CF.log 2>&1
    echo "$V warps=$W $CF rc=$? $(grep -o '"value": [0-9.e+]*' gpurun_out/bsab_${TAG}_${V}_${W}_$CF.log | head -1)"
  done
done
