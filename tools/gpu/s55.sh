# Final check of HEAD after the register-pressure fix: GPU suite, smoke, default bench line, HBM line
mkdir -p gpurun_out/s55
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s55/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s55/pytest_gpu.log; tail -2 gpurun_out/s55/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s55/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s55/smoke.log; tail -2 gpurun_out/s55/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s55/c2_host.json 2> gpurun_out/s55/c2_host.err
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s55/c2_hbm.json 2> gpurun_out/s55/c2_hbm.err
for f in c2_host c2_hbm; do python -c "import json; d=json.loads(open('gpurun_out/s55/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"; done
timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s55/hop.json 2>> gpurun_out/s55/err.log; python -c "import json; d=json.load(open('gpurun_out/s55/hop.json')); print('hop', d['sampler_us_per_batch'], d['hop_graph_us'], d['digest'])"
timeout 1500 python bench.py --config c3 --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/s55/c3_host.json 2> gpurun_out/s55/c3_host.err; python -c "import json; d=json.loads(open('gpurun_out/s55/c3_host.json').read().strip().splitlines()[-1]); print('c3_host', d['value'], d['e2e']['value'], d['roofline']['frac'])"
