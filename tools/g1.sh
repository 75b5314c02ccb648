cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 1500 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g1_smoke.log
timeout 600 python bench.py > gpurun_out/g1_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/g1_bench.log
tail -3 gpurun_out/g1_pytest.log; tail -1 gpurun_out/g1_smoke.log; tail -2 gpurun_out/g1_bench.log | cut -c1-600
