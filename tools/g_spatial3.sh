cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python tools/bench_spatial.py --res 256 --out gpurun_out/spatial_prof.json > gpurun_out/spatial_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/spatial_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('single', d['single_gpu_ms'], d['single_phases_ms'])
for s in d['shards']: print(s['G'], s['max_rank_ms'], s['phases_all_ranks_ms'])"
