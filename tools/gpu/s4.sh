mkdir -p gpurun_out/s4
timeout 900 python -m pytest tests/test_gpu_sampler_paths.py tests/test_gpu_sampler.py tests/test_gpu_c2.py tests/test_gpu_pipeline.py -q > gpurun_out/s4/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4/pytest.log
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s4/hbm.json 2> gpurun_out/s4/hbm.err
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s4/host.json 2> gpurun_out/s4/host.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s4/launches_hbm.csv python tools/profile_step.py --steps 3 --features hbm > gpurun_out/s4/prof.log 2>&1
tail -3 gpurun_out/s4/pytest.log
