# ncu --set full of one K1b launch on C4 (2000 recorded steps, no burn-in)
TAG=${1:-r3c}
mkdir -p gpurun_out
KREGEX=bitslice_kernel bash scripts/profile.sh $TAG --layout 3 --burn-in 0 --window 2000
ls -la gpurun_out/ | tail -5
