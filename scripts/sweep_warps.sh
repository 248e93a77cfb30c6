for W in 32 25 20 16 28; do
  echo -n "W=$W "
  timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --burn-in 0 --window 4000 --warps $W 2>/dev/null | grep -o '"value": [0-9.e+]*' | head -1
done
