mkdir -p gpurun_out
./alt/probe_mixed > gpurun_out/probe_mixed.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
cat gpurun_out/probe_mixed.txt; tail -5 gpurun_out/pytest_gpu.log
for v in 1 0; do CP_STREAM_PREFETCH=$v NSW=50 python tools/time_sweep.py c4a 200; done 2>&1 | tee gpurun_out/prefetch_ab.txt
(cd alt/r01 && NSW=1 python tools/time_sweep.py c4a 200) 2>&1 | tee -a gpurun_out/prefetch_ab.txt
NSW=1 python tools/time_sweep.py c4a 200 2>&1 | tee -a gpurun_out/prefetch_ab.txt
