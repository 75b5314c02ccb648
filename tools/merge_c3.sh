#!/bin/bash
# C3 step with each forward variant choice (gpurun box).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for v in scatter merge measure; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config c3 --variant $v > gpurun_out/mc3_$v.log 2>&1
done
python - <<'PY'
import json
for v in ("scatter", "merge", "measure"):
    try:
        d = json.loads([l for l in open(f"gpurun_out/mc3_{v}.log") if l.startswith("{")][-1])
        print(v, d["ms_per_step"], d["config"]["fwd_variants"], {k: x for k, x in d["kernels"].items() if x > 0.1})
    except Exception as e:
        print(v, "failed", e, open(f"gpurun_out/mc3_{v}.log").read()[-2000:])
PY
