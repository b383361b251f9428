# c3 (256^3, R = 8) evidence: device times (L2 flushed), the ncu launch list of the same script,
# and one ncu --set full capture of the c3 stream kernel (mode-0 MTTKRP + the sweep's passes).
mkdir -p gpurun_out
TAG=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python tools/c3_knobs.py > gpurun_out/${TAG}_c3_times.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches_c3.csv python tools/c3_knobs.py > gpurun_out/${TAG}_ncu_c3_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_mma_kernel -s 6 -c 4 \
  -o gpurun_out/${TAG}_c3_stream python tools/c3_knobs.py > gpurun_out/${TAG}_ncu_c3_full.log 2>&1
cat gpurun_out/${TAG}_c3_times.txt
