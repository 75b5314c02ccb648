cd ${GRAFT_REPO_ROOT:-.}
ARGS="--steps 2 --warmup 1 --no-cpu-baseline --variant scatter"
for K in ${KERNELS:-conv_fwd_kernel conv_bwd_kernel fwd_classify fwd_resolve}; do
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:"$K" -c 1 -o gpurun_out/${TAG:-r01k}_${K} python bench.py $ARGS > /dev/null 2>&1
  echo "$K rc=$?"
done
