# Refresh of the round-1-only lines with the session-3 sampler: papers100M shape with features in HBM, 1B-edge C5 (proximity / random)
mkdir -p gpurun_out/s47
timeout 1800 python bench.py --config c3 --features hbm --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/s47/c3_hbm.json 2> gpurun_out/s47/c3_hbm.err
python -c "import json; d=json.loads(open('gpurun_out/s47/c3_hbm.json').read().strip().splitlines()[-1]); print('c3_hbm', d['value'], d['e2e']['value'], d['roofline']['frac'])"
timeout 1800 python bench.py --config c5 --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/s47/c5_host.json 2> gpurun_out/s47/c5_host.err
python -c "import json; d=json.loads(open('gpurun_out/s47/c5_host.json').read().strip().splitlines()[-1]); print('c5_host', d['value'], d['e2e']['value'], d['roofline']['frac'], d.get('hit_pct'))"
timeout 1800 python bench.py --config c5 --order random --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/s47/c5_random.json 2> gpurun_out/s47/c5_random.err
python -c "import json; d=json.loads(open('gpurun_out/s47/c5_random.json').read().strip().splitlines()[-1]); print('c5_random', d['value'], d['e2e']['value'], d['roofline']['frac'], d.get('hit_pct'))"
for f in gpurun_out/s47/*.err; do tail -n 3 $f; done
