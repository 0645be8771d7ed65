mkdir -p gpurun_out/s17
timeout 1200 python tools/policy_sweep.py --out gpurun_out/s17/policy_sweep_c2.json > gpurun_out/s17/policy_sweep.log 2>&1
tail -45 gpurun_out/s17/policy_sweep.log
