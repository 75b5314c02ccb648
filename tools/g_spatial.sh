cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_spatial_gpu.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/spatial_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/spatial_pytest.log
tail -40 gpurun_out/spatial_pytest.log
