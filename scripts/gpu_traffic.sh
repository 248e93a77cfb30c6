# DRAM traffic of one full-size C4 K1 launch (bench configuration), for bench.py's roofline.traffic
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:traj_kernel -c 1 --csv --log-file gpurun_out/traffic_C4.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/traffic_run.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/traffic_C4.csv | tail -4
