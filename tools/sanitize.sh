#!/bin/bash
# compute-sanitizer over tools/sanitize.py (every C-ABI op, small inputs) with each tool; the
# logs go to gpurun_out/sanitize_<tool>.log (summaries copied under profiles/ by the caller).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for T in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_$T.log 2>&1
  echo "$T rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Error' gpurun_out/sanitize_$T.log | tail -2 | tr '\n' ' ')"
done
