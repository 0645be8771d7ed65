mkdir -p gpurun_out/s2
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s2/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s2/pytest_gpu.log
tail -c 4000 gpurun_out/s2/pytest_gpu.log
