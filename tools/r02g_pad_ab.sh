mkdir -p gpurun_out
for r in 1 2; do for v in head pad8; do
  if [ $v = head ]; then L=paper_1111_6091_b200/lib/libcp.so; else L=alt/$v/libcp.so; fi
  echo "== $v"; CP_LIB_PATH=$PWD/$L python tools/prof_modeprod.py c3 50
  CP_LIB_PATH=$PWD/$L python tools/prof_modeprod.py c4a 10
  for cfg in c4a c4b c3; do echo -n "$v: "; CP_LIB_PATH=$PWD/$L NSW=50 python tools/time_sweep.py $cfg 400; done
done; done 2>&1 | tee gpurun_out/pad_ab.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
