# A/B of library variants on the C4 bench (alternating to cancel drift)
TAG=${1:-ab}; shift
for round in 1 2; do
for v in default "$@"; do
  if [ $v = default ]; then unset PBN_LIB_VARIANT; else export PBN_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_${v}_$round.log 2>&1
  echo "$v round $round: $(tail -1 gpurun_out/bench_${TAG}_${v}_$round.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["kernel_ms_median"])')"
done
done
