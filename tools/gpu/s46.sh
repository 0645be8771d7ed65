# Session-3 final check: full GPU suite, smoke, A/B of the default walk vs the pre-split build, bench lines, launch lists
mkdir -p gpurun_out/s46
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s46/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s46/pytest_gpu.log; tail -2 gpurun_out/s46/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s46/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s46/smoke.log; tail -2 gpurun_out/s46/smoke.log
for i in 1 2; do for v in prev cur; do
if [ $v = cur ]; then unset BGL_LIB_PATH; else export BGL_LIB_PATH=$PWD/tools/ab/libbgl_$v.so; fi
timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s46/hop_${v}_$i.json 2>> gpurun_out/s46/err.log
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s46/c2_hbm_${v}_$i.json 2>> gpurun_out/s46/err.log
done; done
unset BGL_LIB_PATH
for f in gpurun_out/s46/hop_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['sampler_us_per_batch'], d['hop_graph_us'], d['digest'])"; done
for f in gpurun_out/s46/c2_hbm_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'])"; done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s46/c2_host.json 2> gpurun_out/s46/c2_host.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/s46/ref.json 2> gpurun_out/s46/ref.err
for f in c2_host ref; do python -c "import json; d=json.loads(open('gpurun_out/s46/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d.get('e2e',{}).get('value'), d.get('roofline',{}).get('frac'))"; done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s46/launches_c2_hbm.csv python tools/profile_step.py --steps 3 --features hbm > gpurun_out/s46/prof_hbm.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s46/launches_c2_host.csv python tools/profile_step.py --steps 3 > gpurun_out/s46/prof_host.log 2>&1
