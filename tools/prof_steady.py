"""One warm-up call and one cp_als_sweeps(nsw) call on a config (random data) -- the steady-state
sweep loop for ncu:  python tools/prof_steady.py c3 [nsw]   (env SMALL=1: fused/tiny small-tensor path)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402

name = sys.argv[1]
nsw = int(sys.argv[2]) if len(sys.argv) > 2 else 4
if name.startswith("cube"):
    s, R = int(name[4:]), 3
    dims = (s, s, s)
else:
    _, dims, R, *_ = cpsynth.CONFIGS[name]
rng = np.random.default_rng(0)
Zd = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device="cuda")
A = [torch.from_numpy(np.ascontiguousarray(rng.standard_normal((R, I)))).cuda().t() for I in dims]
ws = cp.Workspace(dims, R)
nz = cp.norm2(Zd, dims, ws=ws)
out = torch.empty(4, dtype=torch.float64, device="cuda")
cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws, nsweeps=2)
torch.cuda.synchronize()
cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws, nsweeps=nsw)
torch.cuda.synchronize()
print(name, dims, R, "status", out[2].item(), "launches", cp.last_launch_count())
