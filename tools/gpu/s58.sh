# Final full GPU suite + smoke + default bench line on HEAD
mkdir -p gpurun_out/s58
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s58/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s58/pytest_gpu.log; tail -2 gpurun_out/s58/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s58/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s58/smoke.log; tail -2 gpurun_out/s58/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s58/c2_host.json 2> gpurun_out/s58/c2_host.err
python -c "import json; d=json.loads(open('gpurun_out/s58/c2_host.json').read().strip().splitlines()[-1]); print('c2_host', d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
