mkdir -p gpurun_out
for r in 1 2; do for v in head nopipe; do
  if [ $v = head ]; then L=paper_1111_6091_b200/lib/libcp.so; else L=alt/$v/libcp.so; fi
  for cfg in c4a c4b c3 c1; do echo -n "$v: "; CP_LIB_PATH=$PWD/$L NSW=50 python tools/time_sweep.py $cfg 400; done
done; done 2>&1 | cut -c1-140 | tee gpurun_out/pipe_ab.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
