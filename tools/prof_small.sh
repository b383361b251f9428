mkdir -p gpurun_out
GRAPH=1 timeout 120 python tools/time_sweep.py c4a 200 > gpurun_out/prof_small.log 2>&1
GRAPH=1 timeout 120 python tools/time_sweep.py c2 200 >> gpurun_out/prof_small.log 2>&1
CP_PDL=0 timeout 120 python tools/trace_sweep.py c4a 2 >> gpurun_out/prof_small.log 2>&1
timeout 600 ncu --set full --import-source on --cache-control none --clock-control none -k regex:'ymm|solve|prep' --launch-skip 36 --launch-count 6 -f -o gpurun_out/small_warm python tools/time_sweep.py c4a 10 >> gpurun_out/prof_small.log 2>&1
cat gpurun_out/prof_small.log | grep -v Warn
