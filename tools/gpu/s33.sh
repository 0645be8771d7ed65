# Round-2 session-3 check: full GPU suite, smoke, bench lines (C2 host default, ref arm, C2 HBM, C3 host),
# launch lists, ncu full capture of the hop-3 walk, sanitizer over the sampler modes
mkdir -p gpurun_out/s33/sanitizer
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s33/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s33/pytest_gpu.log
tail -3 gpurun_out/s33/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s33/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s33/smoke.log; tail -2 gpurun_out/s33/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s33/c2_host.json 2> gpurun_out/s33/c2_host.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/s33/ref.json 2> gpurun_out/s33/ref.err
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s33/c2_hbm.json 2> gpurun_out/s33/c2_hbm.err
for f in c2_host c2_hbm ref; do python -c "import json; d=json.loads(open('gpurun_out/s33/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d.get('e2e',{}).get('value'), d.get('roofline',{}).get('frac'))"; done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s33/launches_c2_hbm.csv python tools/profile_step.py --steps 3 --features hbm > gpurun_out/s33/prof_hbm.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s33/launches_c2_host.csv python tools/profile_step.py --steps 3 > gpurun_out/s33/prof_host.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"sample_seg|gather_v4" -c 4 -o gpurun_out/s33/full_c2_hbm python tools/profile_step.py --steps 1 --features hbm > gpurun_out/s33/full_hbm.log 2>&1
for m in "" slice hybrid; do
  tag=${m:-seg}
  BGL_SAMPLER=$m timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py > gpurun_out/s33/sanitizer/racecheck_$tag.txt 2>&1; echo "rc=$?" >> gpurun_out/s33/sanitizer/racecheck_$tag.txt; tail -2 gpurun_out/s33/sanitizer/racecheck_$tag.txt
  BGL_SAMPLER=$m timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > gpurun_out/s33/sanitizer/memcheck_$tag.txt 2>&1; echo "rc=$?" >> gpurun_out/s33/sanitizer/memcheck_$tag.txt; tail -2 gpurun_out/s33/sanitizer/memcheck_$tag.txt
done
timeout 1500 python bench.py --config c3 --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/s33/c3_host.json 2> gpurun_out/s33/c3_host.err
python -c "import json; d=json.loads(open('gpurun_out/s33/c3_host.json').read().strip().splitlines()[-1]); print('c3_host', d['value'], d['e2e']['value'], d['roofline']['frac'])"
