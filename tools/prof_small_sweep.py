"""Fused small-sweep kernel on 4^3 and 25^3 (R = 3), 50 sweeps per launch (for ncu captures)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import cpsynth, paper_1111_6091_b200 as cp
for s in (4, 25):
    dims = (s, s, s); Z, A = cpsynth.random_problem(dims, 3, seed=1)
    Zd = torch.from_numpy(Z).cuda(); Ad = [torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t() for a in A]
    nz = cp.norm2(Zd, dims)
    cp.als_sweep(Zd, dims, Ad, nz, nsweeps=50); torch.cuda.synchronize()
