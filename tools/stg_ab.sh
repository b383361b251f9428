mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps_then_gradient.py tests/test_gpu_mg.py tests/test_gpu_tiny_sweep.py -x -q 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gradient or fused_small or normalized or enotspd" 2>&1 | tail -2
for t in 0 1 0 1; do
  echo "== CP_SWEEPS_GRAD_FUSED=$t"
  CP_SWEEPS_GRAD_FUSED=$t timeout 600 python tools/mg_bench.py c1 - 1e-9 2>&1 | tail -1
  CP_SWEEPS_GRAD_FUSED=$t timeout 600 python tools/mg_bench.py dense100 3 1e-10 2>&1 | tail -1
done 2>&1 | tee gpurun_out/stg_mg.txt | cut -c1-100
