# ncu --set full of the c4b (96^4, R = 10) MTTKRP stream kernel (mode 1 and mode 3), summarized
# on the box (the .ncu-rep stays there); plus the stall breakdown.
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'stream_mma' --launch-skip 2 --launch-count 2 -f -o /tmp/c4b_mttkrp python tools/prof_mttkrp.py c4b 2 1,3 > gpurun_out/ncu_c4b.log 2>&1
python tools/summarize_ncu.py gpurun_out/ncu_c4b_summary.md /tmp/c4b_mttkrp.ncu-rep:c4b_mttkrp > gpurun_out/sum_c4b.log 2>&1
python tools/ncu_stalls.py /tmp/c4b_mttkrp.ncu-rep > gpurun_out/stalls_c4b.txt 2>&1
ncu -i /tmp/c4b_mttkrp.ncu-rep --page details --csv > gpurun_out/c4b_details.csv 2>/dev/null
cat gpurun_out/ncu_c4b_summary.md | head -40; head -40 gpurun_out/stalls_c4b.txt
