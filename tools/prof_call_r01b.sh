set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_mma.json 2> gpurun_out/bench_mma.err || exit 1
tail -1 gpurun_out/bench_mma.json
python bench.py --workload c4b --steps 100 --warmup 5 --no-cpu 2>/dev/null | tail -1
python bench.py --workload c3 --steps 100 --warmup 5 --no-cpu 2>/dev/null | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_bench_mma.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-rows > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:stream_mma --launch-skip 2 --launch-count 2 -f -o gpurun_out/r01_mma_c4a python tools/prof_sweep.py c4a 1 > gpurun_out/ncu_mma_c4a.log 2>&1
ls -la gpurun_out
