mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
VARIANTS="head noall" WITH_R01=1 bash tools/r02g_ab.sh
for cfg in c4b c3 c1; do for lean in 1 0; do echo -n "lean=$lean NSW=50 "; CP_STREAM_LEAN=$lean NSW=50 python tools/time_sweep.py $cfg 400; done; done 2>&1 | tee gpurun_out/lean_ab.txt
for lean in 1 0; do echo -n "lean=$lean NSW=50 "; CP_STREAM_LEAN=$lean NSW=50 NOPROF=1 python tools/time_sweep.py c4a 400; done 2>&1 | tee -a gpurun_out/lean_ab.txt
