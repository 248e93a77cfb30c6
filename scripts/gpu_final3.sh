# evidence pass (round 2, K1b): tests, smoke, every bench line, launch list, DRAM traffic, one ncu --set full of K1b
TAG=${1:-r6z}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_$TAG.log | cut -c1-300
timeout 900 python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_C3_$TAG.log 2>&1; echo "C3 rc=$?"
timeout 900 python bench.py --config C6 --no-cpu-baseline > gpurun_out/bench_C6_$TAG.log 2>&1; echo "C6 rc=$?"
timeout 900 python bench.py --geometric --no-cpu-baseline > gpurun_out/bench_geo_$TAG.log 2>&1; echo "geo rc=$?"
timeout 900 python bench.py --sweep --steps 3 --warmup 3 > gpurun_out/sweep_$TAG.jsonl 2>&1; echo "sweep rc=$?"
timeout 1200 python bench.py --protocol C2,C3 > gpurun_out/protocol_$TAG.jsonl 2>&1; echo "protocol rc=$?"; cut -c1-300 gpurun_out/protocol_$TAG.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:bitslice_kernel -c 1 --csv --log-file gpurun_out/traffic_$TAG.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/traffic_run_$TAG.log 2>&1; echo "traffic rc=$?"; tail -4 gpurun_out/traffic_$TAG.csv
KREGEX=bitslice_kernel bash scripts/profile.sh $TAG --burn-in 0 --window 2000
