# A/B of the segmented-walk variants (separate builds): HEAD, default (lean compare, branchy append, one-pass post), branch-free append, two-pass post
mkdir -p gpurun_out/s27
for i in 1 2; do
for v in head cur bf 2p; do
if [ $v = cur ]; then unset BGL_LIB_PATH; else export BGL_LIB_PATH=$PWD/tools/ab/libbgl_$v.so; fi
timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s27/hop_${v}_$i.json 2>> gpurun_out/s27/hop.err
done; done
unset BGL_LIB_PATH
for f in gpurun_out/s27/hop_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['sampler_us_per_batch'], d['hop_graph_us'], d['digest'])"; done
