# Look-back polls with nanosleep back-off vs the previous build; sampler parity
mkdir -p gpurun_out/s41
timeout 1200 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_sampler_paths.py tests/test_gpu_c1.py tests/test_gpu_c2.py -q > gpurun_out/s41/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s41/pytest.log; tail -3 gpurun_out/s41/pytest.log
for i in 1 2; do
BGL_LIB_PATH=$PWD/tools/ab/libbgl_prev.so timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s41/hop_prev_$i.json 2>> gpurun_out/s41/hop.err
timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s41/hop_cur_$i.json 2>> gpurun_out/s41/hop.err
done
for f in gpurun_out/s41/hop_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['sampler_us_per_batch'], d['hop_graph_us'], d['digest'])"; done
for i in 1 2; do
BGL_LIB_PATH=$PWD/tools/ab/libbgl_prev.so timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s41/c2_hbm_prev_$i.json 2>> gpurun_out/s41/err.log
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s41/c2_hbm_cur_$i.json 2>> gpurun_out/s41/err.log
done
for f in gpurun_out/s41/c2_hbm_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'])"; done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/s41/launches_hbm.csv python tools/profile_step.py --steps 3 --features hbm > gpurun_out/s41/prof.log 2>&1
timeout 600 python tools/seg_timeline.py --config c2 --features hbm --out gpurun_out/s41/seg_timeline.json > gpurun_out/s41/seg_timeline.log 2>&1; grep -o "'parents': [0-9]*\|'setup_split_us_mean': {[^}]*}\|'span_us': [0-9.]*" gpurun_out/s41/seg_timeline.log
