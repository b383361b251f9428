for r in 1 2; do for v in $VARIANTS; do
  if [ $v = head ]; then L=paper_1111_6091_b200/lib/libcp.so; else L=alt/$v/libcp.so; fi
  echo "== $v"; CP_LIB_PATH=$PWD/$L python tools/prof_modeprod.py ${CFG:-c3} 50
done; done 2>&1 | tee gpurun_out/gemm_ab.txt
