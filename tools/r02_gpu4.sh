mkdir -p gpurun_out
T=${TAG:-r02c}
timeout 600 python -m pytest tests/test_gpu_guards.py -q > gpurun_out/${T}_guards.log 2>&1; tail -1 gpurun_out/${T}_guards.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "sweep or ylsolve or gradient or fit" > gpurun_out/${T}_parity.log 2>&1; tail -1 gpurun_out/${T}_parity.log
for c in c4a c3 c4b; do NOPROF=1 timeout 300 python tools/time_sweep.py $c 100; done > gpurun_out/${T}_time_sweep.txt 2>&1; cat gpurun_out/${T}_time_sweep.txt
CP_NVCC_EXTRA="-DCP_CTA_TIMELINE" python -m paper_1111_6091_b200.build --force > /dev/null
for c in c4a c3; do
  NOPROF=1 timeout 300 python tools/time_sweep.py $c 2 > gpurun_out/${T}_tl_$c.log 2>&1
  echo "== $c"; python tools/sweep_timeline.py gpurun_out/${T}_tl_$c.log 7
done
python -m paper_1111_6091_b200.build --force > /dev/null
