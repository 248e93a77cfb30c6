# warps-per-group sweep on C4 (default build) and register-rich builds
for W in 16 20 24 28 32 20; do
  echo -n "default W=$W "; timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --warps $W 2>/dev/null | grep -o '"value": [0-9.e+]*' | head -1
done
export PBN_LIB_VARIANT=libpbnsim_t640.so
for W in 20 16; do echo -n "t640 W=$W "; timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --warps $W 2>/dev/null | grep -o '"value": [0-9.e+]*' | head -1; done
export PBN_LIB_VARIANT=libpbnsim_t768.so
for W in 24 20; do echo -n "t768 W=$W "; timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --warps $W 2>/dev/null | grep -o '"value": [0-9.e+]*' | head -1; done
