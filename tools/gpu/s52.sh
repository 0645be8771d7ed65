# ncu evidence for the final build: launch list (3 serialised C2 HBM steps) and a full capture of the three hop kernels + the fused gather
mkdir -p gpurun_out/s52
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s52/launches_c2_hbm.csv python tools/profile_step.py --steps 3 --features hbm > gpurun_out/s52/prof_hbm.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"sample_seg|gather_v4" -c 4 -o gpurun_out/s52/full_c2_hbm python tools/profile_step.py --steps 1 --features hbm > gpurun_out/s52/full_hbm.log 2>&1
ls -la gpurun_out/s52
