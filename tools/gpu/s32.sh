# Sampler CTA cap sweep in the pipelined C2 HBM step (other branches co-run on the freed SM capacity)
mkdir -p gpurun_out/s32
for c in 0 444 370 296 518; do
for i in 1 2; do BGL_SAMPLER_CTAS=$c timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s32/c2_hbm_c${c}_$i.json 2>> gpurun_out/s32/err.log; python -c "import json; d=json.loads(open('gpurun_out/s32/c2_hbm_c${c}_$i.json').read().strip().splitlines()[-1]); print('c2_hbm ctas=$c', d['value'], d['e2e']['value'])"; done
done
BGL_SAMPLER_CTAS=444 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s32/c2_host_c444.json 2>> gpurun_out/s32/err.log; python -c "import json; d=json.loads(open('gpurun_out/s32/c2_host_c444.json').read().strip().splitlines()[-1]); print('c2_host ctas=444', d['value'], d['e2e']['value'])"
