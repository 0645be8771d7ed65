# Slice sampler round 3: two-pass post, next-slice prefetch; parity + A/B + launch list
mkdir -p gpurun_out/s23
timeout 1200 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_sampler_paths.py tests/test_gpu_c2.py tests/test_gpu_c1.py -q -x > gpurun_out/s23/pytest_sampler.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s23/pytest_sampler.log
tail -3 gpurun_out/s23/pytest_sampler.log
BGL_SAMPLER=seg timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s23/hop_seg.json 2> gpurun_out/s23/hop.err
for S in auto 1024 512; do if [ $S = auto ]; then unset BGL_SLICE_DRAWS; else export BGL_SLICE_DRAWS=$S; fi; timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s23/hop_slice_$S.json 2>> gpurun_out/s23/hop.err; done
unset BGL_SLICE_DRAWS
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s23/launches_hbm.csv python tools/profile_step.py --steps 3 --features hbm > gpurun_out/s23/prof_hbm.log 2>&1
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s23/c2_hbm.json 2> gpurun_out/s23/c2_hbm.err
python -c "import json; d=json.loads(open('gpurun_out/s23/c2_hbm.json').read().strip().splitlines()[-1]); print('c2_hbm', d['value'], d['e2e']['value'], d['roofline']['frac'])"
