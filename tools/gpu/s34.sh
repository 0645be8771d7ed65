# Heavy-parent threshold sweep (CTA kernel for parents above it): small hops / all hops
mkdir -p gpurun_out/s34
for v in "0 0" "256 0" "512 0" "1024 0" "0 1024" "0 512" "512 1024"; do
  set -- $v
  BGL_HEAVY_DEG_SMALL=$1 BGL_HEAVY_DEG=$2 timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s34/hop_s$1_a$2.json 2>> gpurun_out/s34/err.log
  python -c "import json; d=json.load(open('gpurun_out/s34/hop_s$1_a$2.json')); print('small=$1 all=$2', d['sampler_us_per_batch'], d['hop_graph_us'], d['digest'])"
done
