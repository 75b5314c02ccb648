#!/bin/bash
# C2 network step with 1 / 2 backward passes per item (gpurun box).
cd ${GRAFT_REPO_ROOT:-.}
for o in 1 2; do
  SPC_BWD_OCP=$o timeout 300 python tools/bench_c2.py > gpurun_out/c2_ocp$o.log 2>&1
  python - $o <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/c2_ocp{sys.argv[1]}.log").read().strip().splitlines()[-1])
print("OCP", sys.argv[1], d["graph_us_per_step"], d["phases_us_eager"]["conv_bwd"], d["phases_us_eager"].get("scatter_grad"))
PY
done
