# Counter-RNG sampler lines (north_star's Philox sampler) and the 6x6 walk occupancy with the current walk
mkdir -p gpurun_out/s37
timeout 600 python bench.py --features hbm --rng counter --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s37/c2_hbm_counter.json 2> gpurun_out/s37/err.log
timeout 900 python bench.py --rng counter --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s37/c2_host_counter.json 2>> gpurun_out/s37/err.log
for f in c2_hbm_counter c2_host_counter; do python -c "import json; d=json.loads(open('gpurun_out/s37/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'], d['roofline']['frac'])"; done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s37/launches_hbm_counter.csv python tools/profile_step.py --steps 3 --features hbm --rng counter > gpurun_out/s37/prof.log 2>&1
for i in 1 2; do BGL_SEG_OCC=6x6 timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s37/hop_6x6_$i.json 2>> gpurun_out/s37/err.log; timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s37/hop_8x4_$i.json 2>> gpurun_out/s37/err.log; done
for f in gpurun_out/s37/hop_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['sampler_us_per_batch'], d['hop_graph_us'], d['digest'])"; done
