#!/bin/bash
# Variant G slab kernel at C5 50 % for K splits / accumulator counts (gpurun box).
cd ${GRAFT_REPO_ROOT:-.}
for cfg in "0 0" "2 4" "4 2" "4 1" "2 2"; do
  set -- $cfg
  if [ $1 = 0 ]; then unset SPC_GEMM_PARTS; else export SPC_GEMM_PARTS=$1; fi
  export SPC_GEMM_NACC=$2; [ $2 = 0 ] && unset SPC_GEMM_NACC
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_gemm_slab --csv python tools/c5one.py 0.5 gemm 2>/dev/null | grep gpu__time | tail -1 | awk -F'","' -v c="$cfg" '{print "parts/nacc", c, $NF}'
done
