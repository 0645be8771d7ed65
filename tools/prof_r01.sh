set -x
python bench.py --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --steps 200 --warmup 20 --features hbm --no-cpu-baseline > gpurun_out/bench_c2_hbm.json 2>> gpurun_out/bench_c2.err
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_step.py --steps 4 > gpurun_out/launch_run.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"gather_v4|sample_warp" -s 0 -c 4 -o gpurun_out/prof_c2 python tools/profile_step.py --steps 2 > gpurun_out/prof_run.log 2>&1
ls -la gpurun_out
