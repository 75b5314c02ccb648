#!/bin/bash
# ncu --set full of the variant-M main kernel on C3's second layer (gpurun box).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k regex:"conv_fwd_kernel" --launch-skip ${SKIP:-0} -c ${CNT:-2} -o gpurun_out/${TAG:-merge}_c3l2 \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --config c3 --variant ${VAR:-merge} > gpurun_out/${TAG:-merge}_ncu.log 2>&1
echo rc=$?
