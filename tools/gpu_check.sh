#!/bin/bash
# Usage (on the GPU box via gpurun): bash tools/gpu_check.sh [extra pytest -k expr]
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_parity_gpu.py -q -m "gpu and not slow" --timeout 300 -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
if [ -n "$SANITIZE" ]; then
  timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_parity_gpu.py -q -m gpu -p no:cacheprovider -k "$SANITIZE" > gpurun_out/sanitize.log 2>&1; echo "sanitize rc=$?" >> gpurun_out/sanitize.log
fi
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -2 gpurun_out/smoke.log; grep -E "passed|failed|Error|error" gpurun_out/pytest_gpu.log | tail -12; [ -n "$SANITIZE" ] && grep -E "ERROR|Invalid|at 0x|by thread|rc=" gpurun_out/sanitize.log | head -20; tail -c 3000 gpurun_out/bench.log
