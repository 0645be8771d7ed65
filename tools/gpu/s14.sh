mkdir -p gpurun_out/s14
timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_sampler_paths.py tests/test_gpu_c2.py tests/test_gpu_c1.py -x -q > gpurun_out/s14/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s14/pytest.log
BGL_PREP_MIN=1 timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_sampler_paths.py tests/test_gpu_c1.py -x -q > gpurun_out/s14/pytest_prep1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s14/pytest_prep1.log
tail -2 gpurun_out/s14/pytest.log gpurun_out/s14/pytest_prep1.log
for v in "1.0 0.75 8" "0.9 0.8 8" "1.0 0.6 4"; do set -- $v
  BGL_RUN_GAMMA=$1 BGL_RUN_BIG=$2 BGL_RUN_SMALL=$3 python tools/seg_timeline.py --out gpurun_out/s14/tl_$1_$2_$3.json > gpurun_out/s14/tl_$1_$2_$3.log 2>&1
  echo "knobs $v"; grep -v busy gpurun_out/s14/tl_$1_$2_$3.log | tail -1 | cut -c1-250
  BGL_RUN_GAMMA=$1 BGL_RUN_BIG=$2 BGL_RUN_SMALL=$3 timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s14/hbm_$1_$2_$3.json 2> gpurun_out/s14/hbm_$1_$2_$3.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/s14/hbm_$1_$2_$3.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d.get('stages_ms'))"
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s14/launches.csv python tools/profile_step.py --steps 2 --features hbm > gpurun_out/s14/prof.log 2>&1
