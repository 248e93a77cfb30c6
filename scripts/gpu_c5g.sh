for V in default libpbnsim_g896.so libpbnsim_g768.so; do
  if [ "$V" = default ]; then unset PBN_LIB_VARIANT; else export PBN_LIB_VARIANT=$V; fi
  echo -n "$V C5 "; timeout 600 python bench.py --config C5 --chains 16384 --burn-in 0 --window 10000 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -o '"value": [0-9.e+]*' | head -1
done
