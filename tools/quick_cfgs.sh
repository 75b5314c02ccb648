#!/bin/bash
# Quick timing of every workload (gpurun box): C4 kernel table, C3 step, OctNet trunk, C2 network.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
bash tools/ab.sh libspconv
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config c3 > gpurun_out/qc_c3.log 2>&1
timeout 600 python tools/bench_octnet.py --variant measure > gpurun_out/qc_oct.log 2>&1
timeout 300 python tools/bench_c2.py > gpurun_out/qc_c2.log 2>&1
python - <<'PY'
import json
def last(f):
    return json.loads([l for l in open(f) if l.startswith("{")][-1])
d = last("gpurun_out/qc_c3.log")
print("C3", d["ms_per_step"], {k: v for k, v in d["kernels"].items() if v > 0.1})
d = last("gpurun_out/qc_oct.log")
print("OctNet", d["graph_ms_per_step"], {k: v for k, v in d["phases_ms_eager"].items() if v[0] > 0.2})
d = last("gpurun_out/qc_c2.log")
print("C2", d["graph_us_per_step"], {k: v for k, v in d["phases_us_eager"].items() if v[0] > 40})
PY
