set -x
mkdir -p gpurun_out
python tools/prof_sweep.py c4b 2 || exit 1
ncu --set full --import-source on --clock-control none -k regex:stream_mma --launch-skip 2 --launch-count 2 -f -o gpurun_out/r01_mma_c4b python tools/prof_sweep.py c4b 1 > gpurun_out/ncu_mma_c4b.log 2>&1
ncu --set full --clock-control none -k regex:'ymm|yl_fixup|solve|prep' --launch-skip 6 --launch-count 6 -f -o gpurun_out/r01_small_c4a python tools/prof_sweep.py c4a 1 > gpurun_out/ncu_small.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_bench_c4b.csv python bench.py --workload c4b --steps 2 --warmup 3 --no-cpu --no-rows > /dev/null 2>&1
ls -la gpurun_out
