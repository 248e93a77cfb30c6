TAG=${1:-r4c}
export PBN_LIB_VARIANT=libpbnsim_ilv.so
timeout 900 python -m pytest tests/test_bitslice_gpu.py -x -q 2>&1 | tail -2
unset PBN_LIB_VARIANT
timeout 900 python -m pytest tests/test_bitslice_gpu.py -x -q 2>&1 | tail -2
CONFIGS="C4 C3 C5" bash scripts/gpu_bsab2.sh $TAG default:24 libpbnsim_ilv.so:24
