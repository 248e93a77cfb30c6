# C5 chain-count sweep (BASELINE config 5)
timeout 1500 python bench.py --sweep --steps 1 --warmup 1 > gpurun_out/sweep_c5.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep_c5.log | cut -c1-400
