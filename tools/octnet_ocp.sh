#!/bin/bash
# OctNet3 trunk with default / 1-pass backward (gpurun box), scatter timing.
cd ${GRAFT_REPO_ROOT:-.}
python -m pytest tests/test_parity_gpu.py -q -x -m "gpu and not slow" -k "scatter" -p no:cacheprovider 2>&1 | tail -1
for o in def 1; do
  if [ $o = def ]; then unset SPC_BWD_OCP; else export SPC_BWD_OCP=$o; fi
  timeout 600 python tools/bench_octnet.py --variant measure > gpurun_out/oct_$o.log 2>&1
  python - $o <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/oct_{sys.argv[1]}.log").read().strip().splitlines()[-1])
p = d["phases_ms_eager"]
print("OCP", sys.argv[1], d["graph_ms_per_step"], p["conv_bwd"], p["scatter_grad"])
PY
done
