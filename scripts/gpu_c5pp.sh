for V in default libpbnsim_pre.so; do
  if [ "$V" = default ]; then unset PBN_LIB_VARIANT; else export PBN_LIB_VARIANT=$V; fi
  timeout 600 ncu --set full --clock-control none -k regex:traj_kernel -s 1 -c 1 -o gpurun_out/prof_c5_$V \
    python bench.py --config C5 --chains 16384 --burn-in 0 --window 1000 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "$V rc=$?"
done
