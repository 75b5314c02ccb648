# ncu --set full of the streaming-op kernels on the bench_stream_ops workload (gpurun box).
cd ${GRAFT_REPO_ROOT:-.}
for K in ${KERNELS:-pool_tile_kernel row_index_kernel topk_seg_kernel relu_write_kernel}; do
  timeout 600 ncu --set full --import-source on --clock-control none \
    -k regex:"$K" -c ${COUNT:-1} -o gpurun_out/s_${K} python tools/bench_stream_ops.py --iters 1 > gpurun_out/s_${K}.log 2>&1
  echo "$K rc=$?"
done
