cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k regex:"conv_bwd_kernel" -c 1 -o gpurun_out/r02e_conv_bwd python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bwd.log 2>&1
echo "ncu rc=$?"
ls -la gpurun_out/
