# Profiling recipe for one round (run under gpurun on 1 GPU):
#   bash tools/prof_round.sh <tag>
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_c2.csv python tools/profile_step.py --steps 4 > gpurun_out/${TAG}_launch_run.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"gather_v4|sample_warp|lookup_fused|emit_kernel|insert_kernel|hop_scan" -c 12 \
    -o gpurun_out/${TAG}_full_c2 python tools/profile_step.py --steps 1 > gpurun_out/${TAG}_full_run.log 2>&1
ls -la gpurun_out
