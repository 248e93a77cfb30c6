TAG=${1:-r3s}
mkdir -p gpurun_out
CONFIGS="C4 C3 C5" bash scripts/gpu_bsab2.sh $TAG default:28 libpbnsim_t768.so:24
for V in default libpbnsim_t768.so; do
  if [ "$V" = default ]; then unset PBN_LIB_VARIANT; else export PBN_LIB_VARIANT=$V; fi
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:bitslice_kernel -c 1 --csv --log-file gpurun_out/traffic_${TAG}_$V.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "traffic $V rc=$?"; grep -o '"dram__bytes_[a-z]*.sum","byte","[0-9]*"' gpurun_out/traffic_${TAG}_$V.csv
done
