# Look-back anatomy (diagnostic build): windows and polls of the first chain per run
mkdir -p gpurun_out/s56
timeout 600 python tools/seg_timeline.py --config c2 --features hbm --out gpurun_out/s56/seg_timeline.json > gpurun_out/s56/seg_timeline.log 2>&1; grep -o "'parents': [0-9]*\|'setup_split_us_mean': {[^}]*}\|'lookback1_[a-z_]*': \[[^]]*\]\|'lookback_us_p50_p90_max': \[[^]]*\]" gpurun_out/s56/seg_timeline.log; tail -2 gpurun_out/s56/seg_timeline.log
