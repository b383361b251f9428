mkdir -p gpurun_out
timeout 120 python tools/trace_sweep.py c4a 3 > gpurun_out/trace.log 2>&1
CP_SWEEP_SKIP=1 timeout 120 python tools/trace_sweep.py c4a 3 >> gpurun_out/trace.log 2>&1
CP_PDL=0 timeout 120 python tools/trace_sweep.py c4a 3 >> gpurun_out/trace.log 2>&1
cat gpurun_out/trace.log
