set -x
mkdir -p gpurun_out/s1
nvidia-smi --query-gpu=name,memory.total --format=csv > gpurun_out/s1/smi.txt 2>&1
nproc > gpurun_out/s1/nproc.txt; free -g >> gpurun_out/s1/nproc.txt; df -h /dev/shm >> gpurun_out/s1/nproc.txt; lscpu | head -30 >> gpurun_out/s1/nproc.txt; ls /sys/devices/system/node/ >> gpurun_out/s1/nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s1/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s1/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s1/bench.json 2> gpurun_out/s1/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/s1/ref.json 2> gpurun_out/s1/ref.err
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 5 > gpurun_out/s1/bench_g2.json 2> gpurun_out/s1/bench_g2.err
tail -c 3000 gpurun_out/s1/pytest_gpu.log
