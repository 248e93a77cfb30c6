for S in "1 0" "2 0" "2 2000" "2 500"; do
  set -- $S
  echo -n "schedule=$1 chunk=$2 "
  timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --burn-in 0 --window 20000 --schedule $1 --chunk $2 2>&1 | grep -o '"value": [0-9.e+]*\|Error.*' | head -1
done
