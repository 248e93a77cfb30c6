# usage: bash scripts/profile.sh <tag> [bench args...]
TAG=$1; shift
CMD="python bench.py --no-cpu-baseline --steps 1 --warmup 3 $*"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-traj_kernel} -s 3 -c 1 \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/plain_$TAG.log | cut -c1-400
