# Look-back polls as GPU-scope relaxed loads (volatile compiled to system-scope LDG.STRONG.SYS): parity, A/B, timeline, ncu
mkdir -p gpurun_out/s57
timeout 1800 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_sampler_paths.py tests/test_gpu_c2.py tests/test_gpu_cache.py tests/test_gpu_counter.py -q > gpurun_out/s57/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s57/pytest.log; tail -2 gpurun_out/s57/pytest.log
for i in 1 2; do for v in prev cur; do
if [ $v = cur ]; then unset BGL_LIB_PATH; else export BGL_LIB_PATH=$PWD/tools/ab/libbgl_$v.so; fi
timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s57/hop_${v}_$i.json 2>> gpurun_out/s57/err.log
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s57/c2_hbm_${v}_$i.json 2>> gpurun_out/s57/err.log
done; done
unset BGL_LIB_PATH
for f in gpurun_out/s57/hop_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['sampler_us_per_batch'], d['hop_graph_us'], d['dedup_us_mean'], d['digest'])"; done
for f in gpurun_out/s57/c2_hbm_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'])"; done
timeout 600 python tools/seg_timeline.py --config c2 --features hbm --out gpurun_out/s57/seg_timeline.json > gpurun_out/s57/seg_timeline.log 2>&1; grep -o "'parents': [0-9]*\|'setup_split_us_mean': {[^}]*}\|'span_us': [0-9.]*" gpurun_out/s57/seg_timeline.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s57/launches_c2_hbm.csv python tools/profile_step.py --steps 3 --features hbm > gpurun_out/s57/prof_hbm.log 2>&1
