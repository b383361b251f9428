# A/B of the pre-wait Z prefetch (CP_STREAM_PREFETCH) on one box
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep_tail.py tests/test_gpu_guards.py -x -q 2>&1 | tail -3
for c in c4a c3 c2 c1 c4b; do for t in 0 1 0 1; do
  CP_SMALL_SWEEP=0 CP_STREAM_PREFETCH=$t NOPROF=1 NSW=50 timeout 300 python tools/time_sweep.py $c 400
done; for t in 0 1 0 1; do
  CP_SMALL_SWEEP=0 CP_STREAM_PREFETCH=$t NOPROF=1 NSW=1 timeout 300 python tools/time_sweep.py $c 400
done; done 2>&1 | cut -c1-60 | tee gpurun_out/prefetch_ab.txt
