# Round-2 closing evidence: launch lists of the steady-state sweep loops (c3, c4a, c1) and
# ncu --set full captures of their kernels and of the tiny-level kernel.  One GPU, one process per
# capture, each after the same command ran clean without ncu.
mkdir -p gpurun_out
T=${T:-r02h}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${T}_smi.txt 2>&1
for c in c3 c4a c1 cube4; do timeout 300 python tools/prof_steady.py $c 4 || exit 1; done
for c in c3 c4a c1; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_${c}_steady.csv \
    python tools/prof_steady.py $c 4 > gpurun_out/${T}_ncu_launch_$c.log 2>&1
done
# full captures: the last sweeps' kernels (skip the warm-up call's launches)
timeout 900 ncu --set full --clock-control none -k regex:"stream_mma_kernel|ylsolve" -s 10 -c 8 \
  -o gpurun_out/${T}_c3_steady python tools/prof_steady.py c3 4 > gpurun_out/${T}_ncu_c3_full.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"stream_mma_kernel" -s 4 -c 4 \
  -o gpurun_out/${T}_c4a_steady python tools/prof_steady.py c4a 4 > gpurun_out/${T}_ncu_c4a_full.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"tiny_sweep_kernel" -c 1 \
  -o gpurun_out/${T}_tiny python tools/prof_steady.py cube4 50 > gpurun_out/${T}_ncu_tiny_full.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"gemm_dmma_pipe" -s 6 -c 3 \
  -o gpurun_out/${T}_gemm_c3 python tools/modeprod_bench.py > gpurun_out/${T}_ncu_gemm_full.log 2>&1
# the reports exceed gpurun's 64 MiB return limit: keep the raw metric pages (CSV) only
for r in c3_steady c4a_steady tiny gemm_c3; do
  ncu -i gpurun_out/${T}_$r.ncu-rep --page raw --csv > gpurun_out/${T}_${r}_raw.csv 2>/dev/null
  rm -f gpurun_out/${T}_$r.ncu-rep
done
ls -la gpurun_out/ | tail -20
