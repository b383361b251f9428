# round-2 check: build state of the tree on the GPU -- pytest -m gpu, smoke, multigrid trace parity
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02a_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02a_smoke.log
for args in "c0 10 0 u" "c0 10 0 n" "c0 10 1 u" "c0 0 0 u" "c1 0 0 u" "c1 0 1 u" "c1 0 0 n" "c2 25 0 u 30" "c2 25 0 n 30"; do
  timeout 600 python tools/mg_trace_parity.py $args >> gpurun_out/r02a_mg_trace.jsonl 2>> gpurun_out/r02a_mg_trace.err
done
tail -3 gpurun_out/r02a_pytest_gpu.log
