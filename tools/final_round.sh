# End-of-round measurement set (gpurun box): launch list of the bench step, the bench line, the
# network workloads, the streaming ops, smoke.
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r01}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k regex:'spc::' --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --variant scatter > /dev/null 2>&1
echo "launch list rc=$?"
timeout 400 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
timeout 300 python tools/bench_c2.py > gpurun_out/${TAG}_c2.log 2>&1; echo "c2 rc=$?"
timeout 400 python tools/bench_octnet.py --variant measure > gpurun_out/${TAG}_octnet.log 2>&1; echo "octnet rc=$?"
timeout 300 python tools/bench_stream_ops.py --out gpurun_out/${TAG}_stream_ops.json > /dev/null 2>&1; echo "stream rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
