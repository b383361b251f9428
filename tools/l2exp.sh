mkdir -p gpurun_out
for w in c4a c4b c3; do for mb in 0 32 48 64 80 96 112; do CP_L2KEEP_MB=$mb timeout 120 python tools/time_sweep.py $w 200; done; done > gpurun_out/l2exp.log 2>&1
cat gpurun_out/l2exp.log
