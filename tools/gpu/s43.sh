# Look-back with deferred reductions, both chains in lockstep, windows of 32*P runs: P=4 (cur), P=1, previous build
mkdir -p gpurun_out/s43
timeout 1200 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_sampler_paths.py tests/test_gpu_c1.py tests/test_gpu_c2.py -q > gpurun_out/s43/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s43/pytest.log; tail -2 gpurun_out/s43/pytest.log
for i in 1 2; do for v in prev p1 cur; do
if [ $v = cur ]; then unset BGL_LIB_PATH; else export BGL_LIB_PATH=$PWD/tools/ab/libbgl_$v.so; fi
timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s43/hop_${v}_$i.json 2>> gpurun_out/s43/err.log
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s43/c2_hbm_${v}_$i.json 2>> gpurun_out/s43/err.log
done; done
unset BGL_LIB_PATH
for f in gpurun_out/s43/hop_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['sampler_us_per_batch'], d['hop_graph_us'], d['digest'])"; done
for f in gpurun_out/s43/c2_hbm_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'])"; done
timeout 600 python tools/seg_timeline.py --config c2 --features hbm --out gpurun_out/s43/seg_timeline.json > gpurun_out/s43/seg_timeline.log 2>&1; grep -o "'parents': [0-9]*\|'setup_split_us_mean': {[^}]*}\|'lookback_windows_mean_max': [^]]*\]\|'span_us': [0-9.]*" gpurun_out/s43/seg_timeline.log
