# A/B of the in-pass tail solve (CP_SWEEP_TAIL) on one box: parity tests, then ms/sweep.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweep_tail.py -x -q > gpurun_out/tail_tests.log 2>&1; tail -5 gpurun_out/tail_tests.log
for c in c4a c3 c2 c1; do for t in 0 1 2 0 1 2; do
  CP_SMALL_SWEEP=0 CP_SWEEP_TAIL=$t NOPROF=1 NSW=50 timeout 300 python tools/time_sweep.py $c 400
done; for t in 0 2 0 2; do
  CP_SMALL_SWEEP=0 CP_SWEEP_TAIL=$t NOPROF=1 NSW=1 timeout 300 python tools/time_sweep.py $c 400
done; done 2>&1 | cut -c1-48 | tee gpurun_out/tail_ab.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_mg.py -x -q 2>&1 | tail -3
