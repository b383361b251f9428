mkdir -p gpurun_out
CP_NVCC_EXTRA="-DCP_TINY_TIMING" python -m paper_1111_6091_b200.build --force > /dev/null
python - <<'P' 2>&1 | tee gpurun_out/tiny_timing.txt
import numpy as np, torch, cpsynth
import paper_1111_6091_b200 as cp
for s, R in ((4, 3), (5, 3)):
    dims = (s, s, s)
    Z, A = cpsynth.random_problem(dims, R, seed=1)
    Zd = torch.from_numpy(Z).cuda()
    Ad = [torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t() for a in A]
    print("==", dims, R, flush=True)
    cp.als_sweep(Zd, dims, Ad, cp.norm2(Zd, dims), nsweeps=3)
    torch.cuda.synchronize()
P
python -m paper_1111_6091_b200.build --force > /dev/null
timeout 900 python -m pytest tests/test_gpu_tiny_sweep.py -x -q 2>&1 | tail -2
timeout 600 python tools/small_bench.py 2>&1 | head -3
bash tools/tiny_ab.sh 2>&1 | tail -12 | cut -c1-1200
