# compute-sanitizer on every kernel path + warps-per-group sweep on C4
for T in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $T --error-exitcode 9 python scripts/sanitize_run.py > gpurun_out/sanitizer_$T.log 2>&1; echo "$T rc=$?"; tail -3 gpurun_out/sanitizer_$T.log
done
for W in 32 25 20; do
  echo -n "W=$W "; timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --warps $W 2>/dev/null | grep -o '"value": [0-9.e+]*' | head -1
done
