"""Per-call device times of the multigrid's small-level work: cp_als_sweeps (fused vs general
path), cp_gradient, on the c1 level shapes.   python tools/small_bench.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()


def timed(fn, n=20):
    fn()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(n):
        fn()
    e[1].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / n * 1e3  # us


for s, R in ((4, 3), (5, 3), (7, 3), (13, 3), (25, 3), (50, 3), (20, 3), (100, 5)):
    dims = (s, s, s)
    Z, A = cpsynth.random_problem(dims, R, seed=1)
    Zd = torch.from_numpy(Z).cuda()
    Ad = [dev(a) for a in A]
    ws = cp.Workspace(dims, R)
    nz = cp.norm2(Zd, dims, ws=ws)
    row = {"dims": s, "R": R}
    for name, small, tiny in (("tiny", "1", "1"), ("fused", "1", "0"), ("general", "0", "0")):
        if name == "tiny" and s > 5:
            continue
        os.environ["CP_SMALL_SWEEP"] = small
        os.environ["CP_TINY_SWEEP"] = tiny
        A2 = [a.clone() for a in Ad]
        row["sweeps50_" + name] = timed(lambda: cp.als_sweep(Zd, dims, A2, nz, ws=ws, nsweeps=50), n=5)
        row["sweep1_" + name] = timed(lambda: cp.als_sweep(Zd, dims, A2, nz, ws=ws), n=20)
    os.environ["CP_SMALL_SWEEP"] = "1"
    os.environ["CP_TINY_SWEEP"] = "1"
    row["gradient"] = timed(lambda: cp.gradient(Zd, dims, Ad, nz, ws=ws), n=20)
    print({k: (round(v, 1) if isinstance(v, float) else v) for k, v in row.items()})
