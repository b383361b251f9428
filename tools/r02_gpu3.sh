mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_guards.py -q > gpurun_out/r02_guards.log 2>&1; tail -3 gpurun_out/r02_guards.log
# per-CTA timeline of the streaming kernels (CP_CTA_TIMELINE build) on c3 and c4a
CP_NVCC_EXTRA="-DCP_CTA_TIMELINE" python -m paper_1111_6091_b200.build --force > /dev/null
for c in c3 c4a; do
  NOPROF=1 timeout 300 python tools/time_sweep.py $c 2 > gpurun_out/r02_ctl_sweep_$c.log 2>&1
  python tools/cta_timeline.py gpurun_out/r02_ctl_sweep_$c.log
done
timeout 300 python tools/c3_knobs.py > gpurun_out/r02_ctl_c3_mttkrp.log 2>&1
python tools/cta_timeline.py gpurun_out/r02_ctl_c3_mttkrp.log
python -m paper_1111_6091_b200.build --force > /dev/null
# ncu --set full of the c4a sweep's two stream launches
NOPROF=1 timeout 300 python tools/time_sweep.py c4a 3 > gpurun_out/r02_plain_c4a.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_mma_kernel -s 20 -c 2 \
  -o gpurun_out/r02_c4a_stream env NOPROF=1 python tools/time_sweep.py c4a 3 > gpurun_out/r02_ncu_c4a_full.log 2>&1
echo done
