TAG=${1:-r2i}
mkdir -p gpurun_out
for v in default libpbnsim_bsearch.so libpbnsim_inl.so; do
  if [ $v = default ]; then unset PBN_LIB_VARIANT; else export PBN_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --config C6 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C6_${v}_$TAG.log 2>&1; echo "$v rc=$?"
  tail -1 gpurun_out/bench_C6_${v}_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'])"
done
unset PBN_LIB_VARIANT
timeout 600 python -m pytest tests -m gpu -q -x -k "dense or edge_models" > gpurun_out/pytest_dense_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_dense_$TAG.log
