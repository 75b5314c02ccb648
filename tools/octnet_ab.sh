#!/bin/bash
# OctNet3 trunk step for several library builds (gpurun box): bash tools/octnet_ab.sh libA libB ...
cd ${GRAFT_REPO_ROOT:-.}
for L in "$@"; do
  SPC_LIB=paper_1801_10585_b200/$L.so timeout 600 python tools/bench_octnet.py --variant measure > gpurun_out/octab_$L.log 2>&1
  python - $L <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/octab_{sys.argv[1]}.log").read().strip().splitlines()[-1])
p = d["phases_ms_eager"]
print(sys.argv[1], d["graph_ms_per_step"], p["conv_bwd"])
PY
done
