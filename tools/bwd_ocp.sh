#!/bin/bash
# Backward passes-per-item sweep (gpurun box): parity with 1 and 2 passes, C4 / C3 timing.
cd ${GRAFT_REPO_ROOT:-.}
python -m pytest tests/test_parity_gpu.py tests/test_dp_gpu.py -q -x -m "gpu and not slow" -k "bwd or dp or shard" -p no:cacheprovider 2>&1 | tail -1
SPC_BWD_OCP=2 python -m pytest tests/test_parity_gpu.py tests/test_dp_gpu.py -q -x -m "gpu and not slow" -k "bwd or dp or shard" -p no:cacheprovider 2>&1 | tail -1
for o in 1 2; do echo "C4 OCP=$o"; SPC_BWD_OCP=$o bash tools/ab.sh libspconv; done
for o in 1 2; do echo "C3 OCP=$o"; SPC_BWD_OCP=$o timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config c3 2>&1 | grep -o '"ms_per_step": [0-9.]*\|"conv_bwd": {"ms": [0-9.]*'; done
