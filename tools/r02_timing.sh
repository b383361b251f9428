# phase timestamps of the sweep's small kernels (timing build: -DCP_SOLVE_TIMING, globaltimer
# printf per block) on c4a and c3; the stream kernels are unchanged
mkdir -p gpurun_out
bash tools/build_timing.sh
for c in c4a c3; do
  CP_LIB_PATH=$PWD/paper_1111_6091_b200/lib/libcp_timing.so NOPROF=1 timeout 300 python tools/time_sweep.py $c 3 > gpurun_out/r02_timing_$c.log 2>&1
done
python tools/ys_timeline.py gpurun_out/r02_timing_c4a.log; python tools/ys_timeline.py gpurun_out/r02_timing_c3.log
grep "solve mode" gpurun_out/r02_timing_c4a.log | tail -4; grep "solve mode" gpurun_out/r02_timing_c3.log | tail -4
# per-CTA timeline of the streaming kernels (CP_CTA_TIMELINE build) on c3 and c4a
CP_NVCC_EXTRA="-DCP_CTA_TIMELINE" python -m paper_1111_6091_b200.build --force > /dev/null
for c in c3 c4a; do
  NOPROF=1 timeout 300 python tools/time_sweep.py $c 2 > gpurun_out/r02_ctl_sweep_$c.log 2>&1
  python tools/cta_timeline.py gpurun_out/r02_ctl_sweep_$c.log
done
timeout 300 python tools/c3_knobs.py > gpurun_out/r02_ctl_c3_mttkrp.log 2>&1
python tools/cta_timeline.py gpurun_out/r02_ctl_c3_mttkrp.log
python -m paper_1111_6091_b200.build --force > /dev/null
