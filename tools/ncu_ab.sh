#!/bin/bash
# Shared-memory / issue metrics of one kernel for several library builds (gpurun box):
#   KERNEL=conv_fwd_kernel bash tools/ncu_ab.sh libspconv_a libspconv_b ...
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active
for L in "$@"; do
  SPC_LIB=paper_1801_10585_b200/$L.so timeout 600 ncu --metrics $M --clock-control none -k regex:"${KERNEL:-conv_fwd_kernel}" -c 1 --csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --variant scatter --sweep none ${BENCH_ARGS} > gpurun_out/ncuab_$L.csv 2>/dev/null
  echo "== $L"
  python tools/ncu_csv.py gpurun_out/ncuab_$L.csv
done
