#!/bin/bash
# Usage (on the GPU box, via gpurun): bash tools/profile_gpu.sh TAG [KERNEL_REGEX...]
# 1) launch list of every libspconv kernel in a short bench run (gpu__time_duration, serialised)
# 2) one `ncu --set full` capture per kernel regex given
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r01}; shift
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 1 --no-cpu-baseline ${BENCH_ARGS}"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k regex:'spc::' --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py $ARGS > gpurun_out/${TAG}_launches_stdout.log 2>&1
echo "launch list rc=$?"
for K in "$@"; do
  timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:"$K" -c 1 -o gpurun_out/${TAG}_${K} python bench.py $ARGS > gpurun_out/${TAG}_${K}_stdout.log 2>&1
  echo "full capture $K rc=$?"
done
