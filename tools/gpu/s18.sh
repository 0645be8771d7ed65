# full GPU suite + smoke + default bench line + reference arm after the round-2 additions
mkdir -p gpurun_out/s18
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s18/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s18/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s18/smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s18/c2_host.json 2> gpurun_out/s18/c2_host.err
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s18/c2_hbm.json 2> gpurun_out/s18/c2_hbm.err
tail -5 gpurun_out/s18/pytest_gpu.log; cat gpurun_out/s18/smoke.log
for f in c2_host c2_hbm; do python -c "import json; d=json.loads(open('gpurun_out/s18/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'], d['roofline']['frac'], d.get('e2e_dropin',{}).get('value'), d.get('e2e_dropin',{}).get('simulate_ms_per_batch'))"; done
