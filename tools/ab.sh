#!/bin/bash
# A/B timing of library builds (on the GPU box): bash tools/ab.sh libA libB ... (names under
# paper_1801_10585_b200/, without .so). Short bench per build, kernel times printed.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for L in "$@"; do
  SPC_LIB=paper_1801_10585_b200/$L.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --variant scatter --sweep none ${BENCH_ARGS} > gpurun_out/ab_$L.log 2>&1
  python - $L <<'PY'
import json, sys
for l in open("gpurun_out/ab_" + sys.argv[1] + ".log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], d["value"], d["ms_per_step"], {k: v["ms"] for k, v in d["kernels"].items() if v["ms"] > 0.1})
PY
done
