unset PBN_LIB_VARIANT
echo -n "768 W=24 C5 "; timeout 600 python bench.py --config C5 --chains 16384 --burn-in 0 --window 10000 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -o '"value": [0-9.e+]*' | head -1
export PBN_LIB_VARIANT=libpbnsim_g1024.so
for W in 32 24; do echo -n "1024 W=$W C5 "; timeout 600 python bench.py --config C5 --chains 16384 --burn-in 0 --window 10000 --steps 2 --warmup 3 --no-cpu-baseline --warps $W 2>/dev/null | grep -o '"value": [0-9.e+]*' | head -1; done
PBN_FORCE_GLOBAL_IMAGE=1 timeout 300 python scripts/dbg_c2g.py 2>&1 | tail -6
