TAG=${1:-r2l}
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:nodepar -s 1 -c 1 -o gpurun_out/prof_np_C5x64_$TAG python scripts/run_nodelanes.py C5 64 4 1000 2 > gpurun_out/ncu_np_C5x64_$TAG.log 2>&1; echo "ncu rc=$?"
