# generic (dense) path: parent offsets four at a time -- parity and C6
TAG=${1:-r4d}
mkdir -p gpurun_out
export PBN_LIB_VARIANT=libpbnsim_dense.so
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -rf -k "C6 or dense or edge_models or deep_theta or wide_ell or large_configs" > gpurun_out/pytest_dense_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_dense_$TAG.log
unset PBN_LIB_VARIANT
for V in default libpbnsim_dense.so; do
  if [ "$V" = default ]; then unset PBN_LIB_VARIANT; else export PBN_LIB_VARIANT=$V; fi
  timeout 600 python bench.py --config C6 --no-cpu-baseline --e2e-steps 1 --steps 2 > gpurun_out/dense_${TAG}_$V.log 2>&1; echo "$V C6 rc=$? $(grep -o '"value": [0-9.e+]*' gpurun_out/dense_${TAG}_$V.log | head -1)"
done
