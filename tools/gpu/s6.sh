# Round-2 re-entry check: full GPU suite, smoke, C2 host/HBM lines, reference arm, C3 host line + traffic.
mkdir -p gpurun_out/s6
nproc > gpurun_out/s6/host.txt; free -g >> gpurun_out/s6/host.txt; df -h /dev/shm >> gpurun_out/s6/host.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s6/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s6/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6/smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s6/c2_host.json 2> gpurun_out/s6/c2_host.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/s6/ref.json 2> gpurun_out/s6/ref.err
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s6/c2_hbm.json 2> gpurun_out/s6/c2_hbm.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s6/launches_hbm.csv python tools/profile_step.py --steps 3 --features hbm > gpurun_out/s6/prof_hbm.log 2>&1
timeout 1200 python bench.py --config c3 --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/s6/c3_host.json 2> gpurun_out/s6/c3_host.err
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"gather_span|gather_v4|copy_rows" -c 6 -o gpurun_out/s6/full_c3_host python tools/profile_step.py --config c3 --steps 2 --warm 20 > gpurun_out/s6/full_c3.log 2>&1
ls -la gpurun_out/s6
tail -c 1500 gpurun_out/s6/pytest_gpu.log
