# A/B: lockstep double look-back (seg walk) + direct predecessor prefix (dedup emit, cache lookup) vs the affine_cc build
mkdir -p gpurun_out/s29
for i in 1 2; do
BGL_LIB_PATH=$PWD/tools/ab/libbgl_prev.so timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s29/hop_prev_$i.json 2>> gpurun_out/s29/hop.err
timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s29/hop_cur_$i.json 2>> gpurun_out/s29/hop.err
done
for f in gpurun_out/s29/hop_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['sampler_us_per_batch'], d['hop_graph_us'], d['dedup_us_mean'], d['digest'])"; done
BGL_LIB_PATH=$PWD/tools/ab/libbgl_prev.so timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s29/c2_hbm_prev.json 2> gpurun_out/s29/c2_hbm_prev.err
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s29/c2_hbm_cur.json 2> gpurun_out/s29/c2_hbm_cur.err
for f in prev cur; do python -c "import json; d=json.loads(open('gpurun_out/s29/c2_hbm_$f.json').read().strip().splitlines()[-1]); print('c2_hbm $f', d['value'], d['e2e']['value'])"; done
timeout 1200 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_sampler_paths.py tests/test_gpu_cache.py tests/test_gpu_c2.py tests/test_gpu_pipeline.py -q > gpurun_out/s29/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s29/pytest.log; tail -3 gpurun_out/s29/pytest.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s29/launches_hbm.csv python tools/profile_step.py --steps 3 --features hbm > gpurun_out/s29/prof_hbm.log 2>&1
