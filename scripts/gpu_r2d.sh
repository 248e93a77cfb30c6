TAG=${1:-r2d}
mkdir -p gpurun_out
python scripts/run_nodelanes.py C2 1 1 2000 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:nodepar -s 1 -c 1 -o gpurun_out/prof_np_C2_$TAG python scripts/run_nodelanes.py C2 1 1 2000 > gpurun_out/ncu_np_C2_$TAG.log 2>&1; echo "ncu C2 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:nodepar -s 1 -c 1 -o gpurun_out/prof_np_C5_$TAG python scripts/run_nodelanes.py C5 1 8 2000 > gpurun_out/ncu_np_C5_$TAG.log 2>&1; echo "ncu C5 rc=$?"
