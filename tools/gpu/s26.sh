# A/B: look-back walk of the round-2 checkpoint (HEAD build) vs the current walk (lean loop, branch-free append, two-pass post)
mkdir -p gpurun_out/s26
for i in 1 2; do
BGL_LIB_PATH=$PWD/tools/ab/libbgl_head.so timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s26/hop_head_$i.json 2>> gpurun_out/s26/hop.err
timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s26/hop_cur_$i.json 2>> gpurun_out/s26/hop.err
done
BGL_LIB_PATH=$PWD/tools/ab/libbgl_head.so timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s26/c2_hbm_head.json 2> gpurun_out/s26/c2_hbm_head.err
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s26/c2_hbm_cur.json 2> gpurun_out/s26/c2_hbm_cur.err
for f in head cur; do python -c "import json; d=json.loads(open('gpurun_out/s26/c2_hbm_$f.json').read().strip().splitlines()[-1]); print('c2_hbm $f', d['value'], d['e2e']['value'], d['roofline']['frac'])"; done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s26/launches_hbm_cur.csv python tools/profile_step.py --steps 3 --features hbm > gpurun_out/s26/prof_hbm.log 2>&1
