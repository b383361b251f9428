# A/B of stream-kernel variants (alt/<name>/libcp.so, tools/build_variant.py) on c4a, alternating, two rounds
mkdir -p gpurun_out
for round in 1 2; do
  for v in $VARIANTS; do
    if [ $v = head ]; then L=paper_1111_6091_b200/lib/libcp.so; else L=alt/$v/libcp.so; fi
    echo -n "$v: "; CP_LIB_PATH=$PWD/$L NSW=${NSW:-1} python tools/time_sweep.py ${CFG:-c4a} 200
  done
  if [ -n "$WITH_R01" ]; then echo -n "r01: "; (cd alt/r01 && NSW=1 python tools/time_sweep.py ${CFG:-c4a} 200); fi
done 2>&1 | tee gpurun_out/ab_variants.txt
