TAG=${1:-r2c}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rf -x -k "node_lanes" > gpurun_out/pytest_nodelanes_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_nodelanes_$TAG.log
timeout 300 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --csv ./microbench/lds_patterns > gpurun_out/ncu_ldspat_$TAG.csv 2>&1; echo "ncu lds rc=$?"
timeout 600 python scripts/time_fewchain.py C5,C4,C2 2000 > gpurun_out/fewchain_$TAG.jsonl 2>&1; echo "fewchain rc=$?"
PBN_LIB_VARIANT=libpbnsim_acqc.so timeout 600 python scripts/time_fewchain.py C5,C2 2000 > gpurun_out/fewchain_acqc_$TAG.jsonl 2>&1; echo "fewchain acqc rc=$?"
grep node-lanes gpurun_out/fewchain_$TAG.jsonl | cut -c1-150
grep node-lanes gpurun_out/fewchain_acqc_$TAG.jsonl | cut -c1-150
