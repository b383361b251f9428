# tiny (single-warp) sweep kernel: parity tests, per-call times, and the c1 / dense multigrid solves
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tiny_sweep.py -x -q > gpurun_out/tiny_tests.log 2>&1; tail -5 gpurun_out/tiny_tests.log
timeout 600 python tools/small_bench.py 2>&1 | tee gpurun_out/tiny_small_bench.txt
for t in 0 1; do
  echo "== CP_TINY_SWEEP=$t"
  CP_TINY_SWEEP=$t timeout 600 python tools/mg_bench.py c1 - 1e-9 2>&1 | tail -8
  CP_TINY_SWEEP=$t timeout 600 python tools/mg_bench.py dense100 3 1e-10 2>&1 | tail -8
done 2>&1 | tee gpurun_out/tiny_mg.txt
