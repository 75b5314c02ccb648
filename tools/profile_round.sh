#!/bin/bash
# Round profile set (on the GPU box via gpurun): launch list of the bench step, ncu --set full of the
# top C4 kernels, and of variant G on a C5 layer. Usage: bash tools/profile_round.sh TAG
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r01}
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 1 --no-cpu-baseline --variant scatter"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k regex:'spc::' --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py $ARGS > /dev/null 2>&1
echo "launch list rc=$?"
for K in conv_fwd_kernel conv_bwd_kernel fwd_classify fwd_resolve; do
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:"$K" -c 1 -o gpurun_out/${TAG}_${K} python bench.py $ARGS > /dev/null 2>&1
  echo "full capture $K rc=$?"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:conv_gemm_kernel -c 1 \
  -o gpurun_out/${TAG}_conv_gemm_c5 python tools/c5one.py 0.2 gemm > /dev/null 2>&1
echo "full capture conv_gemm rc=$?"
