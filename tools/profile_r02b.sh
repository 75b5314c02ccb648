#!/bin/bash
# End-of-session evidence set, round 2 (on the GPU box): bench lines (C4, C3), launch list of the
# C4 step, ncu --set full of the step's kernels, streaming ops, network steps, C5 sweep, smoke.
# Outputs under gpurun_out/r02b_*.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${TAG:-r02b}
timeout 600 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --config c3 > gpurun_out/${T}_c3.log 2>&1; echo "c3 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k regex:'spc::' --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --variant scatter --sweep none > /dev/null 2>&1
echo "launch list rc=$?"
BENCH_ARGS="--steps 1 --warmup 1 --no-cpu-baseline --variant scatter --sweep none" bash tools/profile_kernels.sh ${T} conv_fwd_kernel conv_bwd_kernel stream_resolve stream_write_kernel conv_fwd_sample row_index_kernel
timeout 600 python tools/bench_stream_ops.py --out gpurun_out/${T}_stream_ops.json > gpurun_out/${T}_stream_ops.log 2>&1; echo "stream ops rc=$?"
timeout 300 python tools/bench_c2.py > gpurun_out/${T}_c2.log 2>&1; echo "c2 rc=$?"
timeout 600 python tools/bench_octnet.py --variant measure > gpurun_out/${T}_octnet.log 2>&1; echo "octnet rc=$?"
timeout 1500 python tools/sweep_c5.py --out gpurun_out/${T}_c5_sweep.jsonl > gpurun_out/${T}_c5.log 2>&1; echo "c5 sweep rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
