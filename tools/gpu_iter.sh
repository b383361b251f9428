# iteration check: GPU parity suite, sweep timings (A/B by env), one timeline
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
for w in c4a c4b c3 c2; do for env in $AB; do env GRAPH=1 $env timeout 120 python tools/time_sweep.py $w 200; done; done > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
CP_PDL=0 timeout 120 python tools/trace_sweep.py c4a 2 2>&1 | grep -v -i warn | tail -20
