#!/bin/bash
# Quick GPU iteration: parity tests (-x), bench (short), optional ncu capture of one kernel.
# Usage: bash tools/quick.sh [ncu-kernel-regex] ; env BENCH_ARGS, PYTEST_K
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -m "gpu and not slow" --timeout 300 -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for ty in ${TY_SWEEP}; do
  SPC_FWD_TY=$ty timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_ty$ty.log 2>&1
  echo "TY=$ty $(grep -o '"conv_fwd": {"ms": [0-9.]*' gpurun_out/bench_ty$ty.log) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_ty$ty.log)"
done
if [ -n "$1" ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$1" -c 1 -o gpurun_out/q_$1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/q_ncu.log 2>&1; echo "ncu rc=$?"
fi
grep -E "passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -3
python - <<'PY'
import json
for l in open("gpurun_out/bench.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("value", d["value"], "ms/step", d["ms_per_step"], "e2e", d.get("e2e", {}).get("value"))
        print({k: v["ms"] for k, v in d["kernels"].items() if v["ms"] > 0.05})
        print("roofline", d["roofline"])
PY
tail -1 gpurun_out/bench.log
