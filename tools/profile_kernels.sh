#!/bin/bash
# ncu --set full captures of the named kernels of the C4 bench step, one report per kernel (on the
# GPU box via gpurun). Usage: bash tools/profile_kernels.sh TAG kernel_regex...
cd ${GRAFT_REPO_ROOT:-.}
TAG=$1; shift
mkdir -p gpurun_out
ARGS=${BENCH_ARGS:-"--steps 1 --warmup 1 --no-cpu-baseline --variant scatter"}
for K in "$@"; do
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:"$K" -c 1 -o gpurun_out/${TAG}_${K} python bench.py $ARGS > gpurun_out/${TAG}_${K}.log 2>&1
  echo "full capture $K rc=$? $(ls -la gpurun_out/${TAG}_${K}.ncu-rep 2>&1)"
done
