mkdir -p gpurun_out/s12
timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_sampler_paths.py tests/test_gpu_c2.py tests/test_gpu_c1.py -x -q > gpurun_out/s12/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s12/pytest.log
tail -3 gpurun_out/s12/pytest.log
for v in "8x4 0.97" "6x6 0.95" "8x4 2.0" "6x6 2.0"; do set -- $v
  BGL_SEG_OCC=$1 BGL_RUN_GAMMA=$2 python tools/seg_timeline.py --out gpurun_out/s12/tl_$1_$2.json > gpurun_out/s12/tl_$1_$2.log 2>&1
  echo "occ $1 gamma $2"; grep -v busy gpurun_out/s12/tl_$1_$2.log | tail -3 | cut -c1-250
  BGL_SEG_OCC=$1 BGL_RUN_GAMMA=$2 timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s12/hbm_$1_$2.json 2> gpurun_out/s12/hbm_$1_$2.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/s12/hbm_$1_$2.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d.get('stages_ms'))"
done
