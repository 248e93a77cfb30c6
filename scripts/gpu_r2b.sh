TAG=${1:-r2b}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rf -x -k "node_lanes" > gpurun_out/pytest_nodelanes_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_nodelanes_$TAG.log
timeout 300 ./microbench/peaks > gpurun_out/peaks_$TAG.json 2> gpurun_out/peaks_$TAG.err; echo "peaks rc=$?"; cat gpurun_out/peaks_$TAG.json
timeout 600 ncu --metrics smsp__inst_executed.sum,sm__cycles_elapsed.max,sm__cycles_elapsed.avg,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,smsp__cycles_active.avg --csv ./microbench/peaks > gpurun_out/ncu_peaks_$TAG.csv 2>&1; echo "ncu peaks rc=$?"
timeout 900 python scripts/time_fewchain.py C5,C4,C2 2000 > gpurun_out/fewchain_$TAG.jsonl 2>&1; echo "fewchain rc=$?"; cat gpurun_out/fewchain_$TAG.jsonl | cut -c1-200
