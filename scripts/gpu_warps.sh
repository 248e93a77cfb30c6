# warps-per-group sweep on C4 (default build)
for W in 16 20 24 28; do
  echo -n "default W=$W "; timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --warps $W 2>/dev/null | grep -o '"value": [0-9.e+]*' | head -1
done
