# Look-back anatomy: windows per chain, first chain time, by run index
mkdir -p gpurun_out/s42
timeout 600 python tools/seg_timeline.py --config c2 --features hbm --out gpurun_out/s42/seg_timeline.json > gpurun_out/s42/seg_timeline.log 2>&1; grep -o "'parents': [0-9]*\|'setup_split_us_mean': {[^}]*}\|'lookback[a-z_]*': [^]]*\]\|'lookback_first_chain_us_mean': [0-9.]*" gpurun_out/s42/seg_timeline.log; tail -3 gpurun_out/s42/seg_timeline.log
