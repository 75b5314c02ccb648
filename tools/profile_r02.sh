#!/bin/bash
# Round-2 evidence set (on the GPU box): launch list of the C4 bench step, ncu --set full of the
# step's kernels, streaming-op table, C5 density sweep. Outputs under gpurun_out/r02_*.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 1 --no-cpu-baseline --variant scatter --sweep none"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k regex:'spc::' --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --variant scatter --sweep none > /dev/null 2>&1
echo "launch list rc=$?"
BENCH_ARGS="--steps 1 --warmup 1 --no-cpu-baseline --variant scatter --sweep none" bash tools/profile_kernels.sh r02 conv_fwd_kernel conv_bwd_kernel stream_resolve stream_write_kernel conv_fwd_sample row_index_kernel
timeout 900 python tools/bench_stream_ops.py --out gpurun_out/r02_stream_ops.json > gpurun_out/r02_stream_ops.log 2>&1; echo "stream ops rc=$?"
timeout 1500 python tools/sweep_c5.py --out gpurun_out/r02_c5_sweep.jsonl > gpurun_out/r02_c5.log 2>&1; echo "c5 sweep rc=$?"
tail -12 gpurun_out/r02_c5.log
