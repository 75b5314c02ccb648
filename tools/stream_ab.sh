#!/bin/bash
# Streaming-op timing for several library builds (gpurun box): bash tools/stream_ab.sh libA libB ...
cd ${GRAFT_REPO_ROOT:-.}
for L in "$@"; do
  echo "== $L"
  SPC_LIB=paper_1801_10585_b200/$L.so timeout 300 python tools/bench_stream_ops.py 2>&1 | grep -v "^{"
done
