# Split-off of long runs' second halves to idle warps: parity (forced splits) + sweep of the split threshold
mkdir -p gpurun_out/s44
timeout 1200 python -m pytest tests/test_gpu_sampler_paths.py -q -k "SPLIT or hubs" > gpurun_out/s44/pytest_paths.log 2>&1; echo "rc=$?" >> gpurun_out/s44/pytest_paths.log; tail -2 gpurun_out/s44/pytest_paths.log
BGL_SEG_SPLIT=64 timeout 1200 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_c1.py tests/test_gpu_c2.py -q > gpurun_out/s44/pytest_split.log 2>&1; echo "rc=$?" >> gpurun_out/s44/pytest_split.log; tail -2 gpurun_out/s44/pytest_split.log
for sp in 0 2048 3072 4096 6144; do BGL_SEG_SPLIT=$sp timeout 600 python tools/hop_bench.py --config c2 --batches 40 --out gpurun_out/s44/hop_sp$sp.json 2>> gpurun_out/s44/err.log; python -c "import json; d=json.load(open('gpurun_out/s44/hop_sp$sp.json')); print('split=$sp', d['sampler_us_per_batch'], d['hop_graph_us'], d['digest'])"; done
tail -3 gpurun_out/s44/err.log
