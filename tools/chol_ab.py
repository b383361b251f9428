"""A/B of the fused small-sweep kernel (cp_als_sweeps, 50 sweeps per call) on coarse-level shapes:
run once per library (CP_LIB_PATH) and compare.   CP_LIB_PATH=... python tools/chol_ab.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()


def timed(fn, n):
    fn()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(n):
        fn()
    e[1].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / n * 1e3  # us


os.environ["CP_SMALL_SWEEP"] = "1"
print("lib", os.environ.get("CP_LIB_PATH", "default"))
for s, R in ((4, 3), (7, 3), (7, 8), (13, 8), (13, 16), (13, 24), (13, 32)):
    dims = (s, s, s)
    Z, A = cpsynth.random_problem(dims, R, seed=1)
    Zd = torch.from_numpy(Z).cuda()
    Ad = [dev(a) for a in A]
    ws = cp.Workspace(dims, R)
    nz = cp.norm2(Zd, dims, ws=ws)
    A2 = [a.clone() for a in Ad]
    t = timed(lambda: cp.als_sweep(Zd, dims, A2, nz, ws=ws, nsweeps=50), n=5)
    print({"dims": s, "R": R, "us_per_sweep": round(t / 50, 2)})
