"""cp_als_sweeps on a medium tensor with the opt-in fused medium kernel (for ncu captures).
    python tools/prof_medium.py [s] [R] [nsweeps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402

os.environ["CP_MEDIUM_SWEEP"] = "1"
s = int(sys.argv[1]) if len(sys.argv) > 1 else 100
R = int(sys.argv[2]) if len(sys.argv) > 2 else 5
nu = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dims = (s, s, s)
Z, A = cpsynth.random_problem(dims, R, seed=1)
Zd = torch.from_numpy(Z).cuda()
Ad = [torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t() for a in A]
nz = cp.norm2(Zd, dims)
for _ in range(2):
    cp.als_sweep(Zd, dims, Ad, nz, nsweeps=nu)
torch.cuda.synchronize()
