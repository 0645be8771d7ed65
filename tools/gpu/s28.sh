# A/B affine_cc walk step vs the previous build, then the full GPU suite + smoke + bench lines
mkdir -p gpurun_out/s28
for i in 1 2; do
BGL_LIB_PATH=$PWD/tools/ab/libbgl_prev.so timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s28/hop_prev_$i.json 2>> gpurun_out/s28/hop.err
timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s28/hop_cur_$i.json 2>> gpurun_out/s28/hop.err
done
for f in gpurun_out/s28/hop_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['sampler_us_per_batch'], d['hop_graph_us'], d['digest'])"; done
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s28/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s28/pytest_gpu.log
tail -3 gpurun_out/s28/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s28/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s28/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s28/c2_host.json 2> gpurun_out/s28/c2_host.err
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s28/c2_hbm.json 2> gpurun_out/s28/c2_hbm.err
for f in c2_host c2_hbm; do python -c "import json; d=json.loads(open('gpurun_out/s28/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'], d['roofline']['frac'])"; done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s28/launches_hbm.csv python tools/profile_step.py --steps 3 --features hbm > gpurun_out/s28/prof_hbm.log 2>&1
