# prep-kernel sampler: parity (sampler goldens, forced overflow paths, C2 window, pipeline), timeline, HBM/host bench
mkdir -p gpurun_out/s10
timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_sampler_paths.py tests/test_gpu_c2.py tests/test_gpu_pipeline.py tests/test_gpu_c1.py -x -q > gpurun_out/s10/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s10/pytest.log
python tools/seg_timeline.py --out gpurun_out/s10/seg_timeline.json > gpurun_out/s10/seg_timeline.log 2>&1
for r in 32; do BGL_RUNS_PER_SM=$r timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s10/hbm_r$r.json 2> gpurun_out/s10/hbm_r$r.err; done
tail -3 gpurun_out/s10/pytest.log
grep -v busy gpurun_out/s10/seg_timeline.log | tail -3
for f in gpurun_out/s10/hbm_*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d.get('stages_ms'))"; done
