# Session-3 final evidence: GPU tests, smoke, default bench (+ reference arm), ncu launch list of
# the bench command, ncu --set full of the c4b MTTKRP stream kernel (tensor-map stage loads).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01s3b_launches_bench_c4a.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-rows > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'stream_mma' --launch-skip 2 --launch-count 2 -f -o /tmp/c4b_tmap python tools/prof_mttkrp.py c4b 2 1,3 > gpurun_out/ncu_c4b.log 2>&1
python tools/summarize_ncu.py gpurun_out/r01s3_ncu_c4b_tmap.md /tmp/c4b_tmap.ncu-rep:c4b_mttkrp_tmap > gpurun_out/sum_c4b.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; head -c 300 gpurun_out/bench.json; cat gpurun_out/r01s3_ncu_c4b_tmap.md
