# Seeds marked before hop 0 and the previous batch's marks cleared there (lazy reset): dedup on the last-hop branch is emit only
mkdir -p gpurun_out/s30
timeout 1500 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_sampler_paths.py tests/test_gpu_c1.py tests/test_gpu_c2.py tests/test_gpu_pipeline.py tests/test_gpu_sharded_pipeline.py tests/test_gpu_counter.py tests/test_gpu_acceptance.py -q > gpurun_out/s30/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s30/pytest.log; tail -3 gpurun_out/s30/pytest.log
for i in 1 2 3; do timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s30/c2_hbm_$i.json 2> gpurun_out/s30/c2_hbm_$i.err; python -c "import json; d=json.loads(open('gpurun_out/s30/c2_hbm_$i.json').read().strip().splitlines()[-1]); print('c2_hbm', d['value'], d['e2e']['value'])"; done
timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s30/hop_cur.json 2>> gpurun_out/s30/hop.err
