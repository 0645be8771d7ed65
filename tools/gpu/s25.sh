# Hybrid walk (lane walk for deg <= 64, slices for the rest): parity + A/B + launch list + C2 HBM line
mkdir -p gpurun_out/s25
timeout 1200 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_sampler_paths.py tests/test_gpu_c2.py tests/test_gpu_c1.py -q > gpurun_out/s25/pytest_sampler.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s25/pytest_sampler.log
tail -5 gpurun_out/s25/pytest_sampler.log
BGL_SAMPLER=seg timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s25/hop_seg.json 2> gpurun_out/s25/hop.err
for D in 64 32 128; do BGL_LANE_DEG=$D timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s25/hop_hyb_$D.json 2>> gpurun_out/s25/hop.err; done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s25/launches_hbm.csv python tools/profile_step.py --steps 3 --features hbm > gpurun_out/s25/prof_hbm.log 2>&1
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s25/c2_hbm.json 2> gpurun_out/s25/c2_hbm.err
python -c "import json; d=json.loads(open('gpurun_out/s25/c2_hbm.json').read().strip().splitlines()[-1]); print('c2_hbm', d['value'], d['e2e']['value'], d['roofline']['frac'])"
