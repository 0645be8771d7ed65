mkdir -p gpurun_out/s3
timeout 900 python -m pytest tests/test_gpu_bench_contract.py tests/test_gpu_sampler_paths.py tests/test_gpu_sampler.py tests/test_gpu_cache.py -q > gpurun_out/s3/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3/pytest.log
for ilp in 1 0; do for bulk in 1 0; do
  BGL_SEG_ILP=$ilp BGL_COPY_BULK=$bulk timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s3/hbm_ilp${ilp}_bulk${bulk}.json 2> gpurun_out/s3/hbm_ilp${ilp}_bulk${bulk}.err
done; done
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s3/host.json 2> gpurun_out/s3/host.err
for ilp in 1 0; do
  BGL_SEG_ILP=$ilp timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s3/launches_hbm_ilp${ilp}.csv python tools/profile_step.py --steps 3 --features hbm > gpurun_out/s3/prof_ilp${ilp}.log 2>&1
done
tail -3 gpurun_out/s3/pytest.log
