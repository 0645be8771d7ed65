# Setup-phase split of the segmented walk (loads / look-back / layout) at C2 HBM
mkdir -p gpurun_out/s39
timeout 600 python tools/seg_timeline.py --config c2 --features hbm --out gpurun_out/s39/seg_timeline.json > gpurun_out/s39/seg_timeline.log 2>&1; cat gpurun_out/s39/seg_timeline.log | tail -8
