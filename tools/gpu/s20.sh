# compute-sanitizer over every kernel family incl. the round-2 ones; ncu full capture of the C2 miss gather
mkdir -p gpurun_out/s20/sanitizer
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > gpurun_out/s20/sanitizer/$t.txt 2>&1; echo "rc=$?" >> gpurun_out/s20/sanitizer/$t.txt
  tail -3 gpurun_out/s20/sanitizer/$t.txt
done
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"gather_span|gather_v4|copy_rows|lookup_fused" -c 4 -o gpurun_out/s20/full_c2_host python tools/profile_step.py --steps 1 > gpurun_out/s20/full_c2_host.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s20/launches_c2_host.csv python tools/profile_step.py --steps 3 > gpurun_out/s20/launch.log 2>&1
ls gpurun_out/s20
