# ncu of the C5 launches: K1 with the image through L1/L2 (16384 chains) and K1c clusters (1024 chains)
python bench.py --config C5 --chains 16384 --burn-in 0 --window 300 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c5a.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traj_kernel -s 3 -c 1 -o gpurun_out/prof_c5k1 \
  python bench.py --config C5 --chains 16384 --burn-in 0 --window 300 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c5a.log 2>&1; echo "k1 rc=$?"
python bench.py --config C5 --chains 1024 --burn-in 0 --window 300 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c5b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traj_cluster -s 3 -c 1 -o gpurun_out/prof_c5k1c \
  python bench.py --config C5 --chains 1024 --burn-in 0 --window 300 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c5b.log 2>&1; echo "k1c rc=$?"
