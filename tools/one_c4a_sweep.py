"""Two c4a sweeps (the second one's prints are the warm ones): for instrumented builds
(CP_LIB_PATH=alt/timing/libcp.so: producer / consumer wait clocks of CTAs 0 and 101)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1111_6091_b200 as cp
dims, R = (512, 512, 512), 16
rng = np.random.default_rng(0)
Z = torch.randn(dims, dtype=torch.float64, device="cuda")
A = [torch.from_numpy(np.ascontiguousarray(rng.standard_normal((R, I)))).cuda().t() for I in dims]
ws = cp.Workspace(dims, R)
nz = cp.norm2(Z, dims, ws=ws)
out = torch.empty(4, dtype=torch.float64, device="cuda")
for i in range(2):
    print(f"--- sweep {i}", flush=True)
    cp.als_sweep(Z, dims, A, nz, out=out, ws=ws)
    torch.cuda.synchronize()
