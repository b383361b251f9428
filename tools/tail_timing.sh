# phase timestamps of the in-pass tail solve (CP_TAIL_TIMING build), c4a and c3, 2 sweeps each
mkdir -p gpurun_out
CP_NVCC_EXTRA="-DCP_TAIL_TIMING" python -m paper_1111_6091_b200.build --force > /dev/null
for c in c4a c3; do echo "== $c"; NOPROF=1 NSW=1 timeout 300 python tools/time_sweep.py $c 1 2>&1 | grep -v "^c[34]" | tail -24; done | tee gpurun_out/tail_timing.txt
python -m paper_1111_6091_b200.build --force > /dev/null
