for V in default libpbnsim_pre.so; do
  if [ "$V" = default ]; then unset PBN_LIB_VARIANT; else export PBN_LIB_VARIANT=$V; fi
  timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,launch__block_size,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:traj_kernel -s 1 -c 1 --csv \
    python bench.py --config C5 --chains 16384 --burn-in 0 --window 2000 --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | grep -E "inst_executed|duration|block_size|issue|hit_rate" | awk -F'","' '{print "'$V' " $(NF-2) " " $NF}'
done
