mkdir -p gpurun_out/s13
for v in "8x4 0.97" "6x6 0.95" "8x4 3.0"; do set -- $v
BGL_SEG_OCC=$1 BGL_RUN_GAMMA=$2 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/s13/launches_$1_$2.csv python tools/profile_step.py --steps 2 --features hbm > gpurun_out/s13/prof_$1_$2.log 2>&1
done
ls gpurun_out/s13
