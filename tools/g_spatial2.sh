cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_spatial_gpu.py -q -x -p no:cacheprovider > gpurun_out/spatial_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/spatial_pytest.log
tail -2 gpurun_out/spatial_pytest.log
timeout 900 python tools/bench_spatial.py --res 256 --out gpurun_out/spatial_r02e.json > gpurun_out/spatial_bench.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/spatial_bench.log | cut -c1-1500
for T in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_$T.log 2>&1
  echo "$T rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Error' gpurun_out/sanitize_$T.log | tail -2 | tr '\n' ' ')"
done
