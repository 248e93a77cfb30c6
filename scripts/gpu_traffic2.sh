# DRAM bytes of the C4 K1b launch: repeatability, and with / without the persistent schedule
TAG=${1:-r3u}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bitslice_gpu.py -x -q -rf > gpurun_out/pytest_bs_$TAG.log 2>&1; echo "pytest bs rc=$?"; tail -2 gpurun_out/pytest_bs_$TAG.log
for i in 1 2 3; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:bitslice_kernel -c 1 --csv --log-file gpurun_out/traffic_${TAG}_p$i.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  echo "persistent $i: $(grep -o '"\(dram__bytes_[a-z]*\|lts__t_bytes\).sum","[a-z]*byte","[0-9.]*"' gpurun_out/traffic_${TAG}_p$i.csv | tr '\n' ' ')"
done
for i in 1 2; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:bitslice_kernel -c 1 --csv --log-file gpurun_out/traffic_${TAG}_s$i.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 --schedule 1 > /dev/null 2>&1
  echo "one unit per group $i: $(grep -o '"\(dram__bytes_[a-z]*\|lts__t_bytes\).sum","[a-z]*byte","[0-9.]*"' gpurun_out/traffic_${TAG}_s$i.csv | tr '\n' ' ')"
done
