cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -x -m gpu -p no:cacheprovider --timeout 900 > gpurun_out/res_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/res_pytest.log
tail -3 gpurun_out/res_pytest.log
timeout 900 python tools/bench_spatial.py --res 256 --out gpurun_out/spatial_r02f.json > gpurun_out/spatial_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/spatial_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('single', d['single_gpu_ms'], d['single_phases_ms'])
for s in d['shards']: print(s['G'], s['max_rank_ms'], s['parity'])"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/res_bench.log 2>&1; echo "c4 rc=$?"; grep -o '"ms_per_step": [0-9.]*' gpurun_out/res_bench.log
