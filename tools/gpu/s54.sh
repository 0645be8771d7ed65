# Final build: full ncu capture of the hop kernels + fused gather; split-off re-check on the fixed walk
mkdir -p gpurun_out/s54
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"sample_seg|gather_v4" -c 4 -o gpurun_out/s54/full_c2_hbm python tools/profile_step.py --steps 1 --features hbm > gpurun_out/s54/full_hbm.log 2>&1
for sp in 0 3072; do for i in 1 2; do BGL_SEG_SPLIT=$sp timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s54/hop_sp${sp}_$i.json 2>> gpurun_out/s54/err.log; BGL_SEG_SPLIT=$sp timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s54/c2_hbm_sp${sp}_$i.json 2>> gpurun_out/s54/err.log; done; done
for f in gpurun_out/s54/hop_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['sampler_us_per_batch'], d['hop_graph_us'])"; done
for f in gpurun_out/s54/c2_hbm_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'])"; done
