# contribution of each launch class to the c4a / c3 sweep time (CP_SWEEP_SKIP drops launches; results wrong)
for c in c4a c3; do
  for sk in 0 1 4 8 16 28 29 128 256 384; do
    echo "$c skip=$sk :: $(CP_SWEEP_SKIP=$sk NOPROF=1 python tools/time_sweep.py $c 2>&1 | tail -1 | cut -c1-90)"
  done
done
