mkdir -p gpurun_out/s5
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s5/c2_host.json 2> gpurun_out/s5/c2_host.err
timeout 600 python bench.py --features hbm --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/s5/c2_hbm.json 2> gpurun_out/s5/c2_hbm.err
timeout 1200 python bench.py --config c3 --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/s5/c3_host.json 2> gpurun_out/s5/c3_host.err
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"gather_span|gather_v4|copy_rows" -c 6 -o gpurun_out/s5/full_c3_host python tools/profile_step.py --config c3 --steps 2 --warm 20 > gpurun_out/s5/full_c3.log 2>&1
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5/launches_c3_host.csv python tools/profile_step.py --config c3 --steps 4 --warm 20 > gpurun_out/s5/launch_c3.log 2>&1
ls -la gpurun_out/s5
