#!/bin/bash
# Bench under several environment settings (on the GPU box): bash tools/envsweep.sh "A=1" "B=2 C=3" ...
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
i=0
for E in "$@"; do
  i=$((i+1))
  env $E timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --variant scatter --sweep none ${BENCH_ARGS} > gpurun_out/env_$i.log 2>&1
  python - "$E" $i <<'PY'
import json, sys
for l in open("gpurun_out/env_" + sys.argv[2] + ".log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], d["value"], d["ms_per_step"], {k: v["ms"] for k, v in d["kernels"].items() if v["ms"] > 0.1})
PY
done
