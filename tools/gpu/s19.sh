mkdir -p gpurun_out/s19
timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_sampler_paths.py tests/test_gpu_c2.py tests/test_gpu_c1.py -x -q > gpurun_out/s19/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s19/pytest.log
tail -2 gpurun_out/s19/pytest.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_fma.sum,smsp__inst_executed_pipe_alu.sum --clock-control none --csv --log-file gpurun_out/s19/launches.csv python tools/profile_step.py --steps 2 --features hbm > gpurun_out/s19/prof.log 2>&1
for i in 1 2; do timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s19/hbm_$i.json 2> gpurun_out/s19/hbm_$i.err
python -c "import json; d=json.loads(open('gpurun_out/s19/hbm_$i.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['stages_ms'])"; done
