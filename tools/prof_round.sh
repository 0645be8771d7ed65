# Profiling recipe for one round (run under gpurun on 1 GPU):
#   bash tools/prof_round.sh <tag> [host|hbm]
set -x
TAG=${1:-r01}
FEAT=${2:-host}
mkdir -p gpurun_out
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_c2_${FEAT}.csv python tools/profile_step.py --steps 4 --features ${FEAT} \
    > gpurun_out/${TAG}_launch_run_${FEAT}.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"gather_v4|gather_list|gather_span|sample_seg|sample_cand|sample_heavy|lookup_fused|emit_kernel|insert_kernel|copy_rows" -c 16 \
    -o gpurun_out/${TAG}_full_c2_${FEAT} python tools/profile_step.py --steps 1 --features ${FEAT} \
    > gpurun_out/${TAG}_full_run_${FEAT}.log 2>&1
ls -la gpurun_out
