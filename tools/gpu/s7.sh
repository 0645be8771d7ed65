# sparse-ID parity + cache regression; sampler occupancy / run-length A/B (HBM features); source-level ncu of the walk
mkdir -p gpurun_out/s7
timeout 900 python -m pytest tests/test_gpu_sparse_ids.py tests/test_gpu_cache.py tests/test_gpu_sharded_pipeline.py -q > gpurun_out/s7/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s7/pytest.log
for v in "8x4 32" "6x6 32" "8x4 48" "8x4 24" "6x6 40"; do set -- $v
  BGL_SEG_OCC=$1 BGL_RUNS_PER_SM=$2 timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s7/hbm_$1_$2.json 2> gpurun_out/s7/hbm_$1_$2.err
done
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:sample_seg -c 3 -o gpurun_out/s7/seg_src python tools/profile_step.py --steps 1 --features hbm > gpurun_out/s7/seg_src.log 2>&1
tail -3 gpurun_out/s7/pytest.log
for f in gpurun_out/s7/hbm_*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d.get('stages_ms'))"; done
