mkdir -p gpurun_out/s11
timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_sampler_paths.py tests/test_gpu_c2.py tests/test_gpu_pipeline.py tests/test_gpu_c1.py -x -q > gpurun_out/s11/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s11/pytest.log
tail -3 gpurun_out/s11/pytest.log
for g in 1.0 1.5 2.0 3.0; do
  BGL_RUN_GAMMA=$g python tools/seg_timeline.py --out gpurun_out/s11/seg_timeline_g$g.json > gpurun_out/s11/seg_timeline_g$g.log 2>&1
  echo "gamma $g"; grep -v busy gpurun_out/s11/seg_timeline_g$g.log | tail -3 | cut -c1-330
  BGL_RUN_GAMMA=$g timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s11/hbm_g$g.json 2> gpurun_out/s11/hbm_g$g.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/s11/hbm_g$g.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d.get('stages_ms'))"
done
