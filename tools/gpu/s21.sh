# Slice sampler (prep + slice walk) first check: sampler parity, A/B hop timing vs the look-back walk, launch list, C2 HBM line
mkdir -p gpurun_out/s21
timeout 1200 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_sampler_paths.py tests/test_gpu_c2.py tests/test_gpu_c1.py -x -q > gpurun_out/s21/pytest_sampler.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s21/pytest_sampler.log
tail -3 gpurun_out/s21/pytest_sampler.log
BGL_SAMPLER=seg timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s21/hop_seg.json 2> gpurun_out/s21/hop_seg.err
timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s21/hop_slice.json 2> gpurun_out/s21/hop_slice.err
for S in 512 2048 4096; do BGL_SLICE_DRAWS=$S timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s21/hop_slice_$S.json 2>> gpurun_out/s21/hop_slice.err; done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s21/launches_hbm.csv python tools/profile_step.py --steps 3 --features hbm > gpurun_out/s21/prof_hbm.log 2>&1
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s21/c2_hbm.json 2> gpurun_out/s21/c2_hbm.err
tail -c 600 gpurun_out/s21/c2_hbm.json
