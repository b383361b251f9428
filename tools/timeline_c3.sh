mkdir -p gpurun_out
CP_NVCC_EXTRA="-DCP_CTA_TIMELINE -DCP_CTA_TIMELINE_STREAM" python -m paper_1111_6091_b200.build --force > /dev/null
for c in c3 c4a; do
  NOPROF=1 NSW=3 timeout 300 python tools/time_sweep.py $c 3 > gpurun_out/tl_$c.log 2>&1
  echo "== $c"; python tools/sweep_timeline.py gpurun_out/tl_$c.log 10
  python tools/cta_timeline.py gpurun_out/tl_$c.log 2>/dev/null | tail -12
done
python -m paper_1111_6091_b200.build --force > /dev/null
