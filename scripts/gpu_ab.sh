# A/B of library variants: parity (GPU tests) + bench + short ncu capture per variant
# usage: bash scripts/gpu_ab.sh <tag> <variant.so[:warps]> ...   ("default" = libpbnsim.so)
TAG=$1; shift
for VW in "$@"; do
  V=${VW%%:*}; W=0; [ "$V" != "$VW" ] && W=${VW##*:}
  if [ "$V" = default ]; then unset PBN_LIB_VARIANT; else export PBN_LIB_VARIANT=$V; fi
  echo "== $V warps=$W"
  timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -k "C1_all or C2_all or large_configs or edge_models" > gpurun_out/pytest_${TAG}_$V.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_${TAG}_$V.log
  timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --warps $W > gpurun_out/bench_${TAG}_$V.log 2>&1; echo "bench rc=$?"
  grep -o '"value": [0-9.e+]*, "unit": "node-updates/s", "n_gpus"' gpurun_out/bench_${TAG}_$V.log | head -1
  [ -n "$PROFILE" ] && { bash scripts/profile.sh ${TAG}_$V --burn-in 0 --window 2000 --warps $W > /dev/null 2>&1; echo "profile rc=$?"; }
done
