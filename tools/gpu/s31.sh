# Branch timeline of the pipelined C2 HBM step, seed-mark placement A/B
mkdir -p gpurun_out/s31
for em in 1 0; do
BGL_EARLY_MARK=$em timeout 600 python tools/branch_timeline.py --config c2 --features hbm --steps 30 --out gpurun_out/s31/branches_hbm_em$em.json 2>> gpurun_out/s31/err.log
BGL_EARLY_MARK=$em timeout 600 python tools/branch_timeline.py --config c2 --features host --steps 30 --out gpurun_out/s31/branches_host_em$em.json 2>> gpurun_out/s31/err.log
for i in 1 2; do BGL_EARLY_MARK=$em timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s31/c2_hbm_em${em}_$i.json 2>> gpurun_out/s31/err.log; python -c "import json; d=json.loads(open('gpurun_out/s31/c2_hbm_em${em}_$i.json').read().strip().splitlines()[-1]); print('c2_hbm em$em', d['value'], d['e2e']['value'])"; done
done
tail -5 gpurun_out/s31/err.log
