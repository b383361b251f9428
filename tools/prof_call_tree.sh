set -x
mkdir -p gpurun_out
python tools/prof_sweep.py c4a 3 && python tools/prof_sweep.py c4b 3 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launch_tree_c4a.csv python tools/prof_sweep.py c4a 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launch_tree_c4b.csv python tools/prof_sweep.py c4b 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:stream_kernel --launch-skip 2 --launch-count 2 -f -o gpurun_out/r01_tree_c4a python tools/prof_sweep.py c4a 1 > gpurun_out/ncu_tree_c4a.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:stream_kernel --launch-skip 2 --launch-count 2 -f -o gpurun_out/r01_tree_c4b python tools/prof_sweep.py c4b 1 > gpurun_out/ncu_tree_c4b.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:'ymm|yl_fixup|yr_kernel|solve|prep|final|reduce' --launch-skip 10 --launch-count 10 -f -o gpurun_out/r01_tree_small_c4a python tools/prof_sweep.py c4a 1 > gpurun_out/ncu_tree_small.log 2>&1
ls -la gpurun_out
