# Candidate-threshold margin sweep with the current walk (branch-free append: the walk's cost no longer depends on it)
mkdir -p gpurun_out/s50
for m in "2,1" "1.5,1" "1,1" "2.5,1" "1.5,0.5"; do BGL_MARGIN=$m timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s50/hop_$m.json 2>> gpurun_out/s50/err.log; python -c "import json; d=json.load(open('gpurun_out/s50/hop_$m.json')); print('margin=$m', d['sampler_us_per_batch'], d['hop_graph_us'], d['digest'])"; done
