mkdir -p gpurun_out/s16
timeout 1200 python -m pytest tests/test_gpu_ordered.py tests/test_gpu_cache.py tests/test_gpu_sparse_ids.py -x -q > gpurun_out/s16/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s16/pytest.log
tail -30 gpurun_out/s16/pytest.log
