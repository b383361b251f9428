"""Run a few sweeps of a config (for printf-instrumented builds):  python tools/one_sweep.py c4a [n]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402

name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
_, dims, R, *_ = cpsynth.CONFIGS[name]
rng = np.random.default_rng(0)
Zd = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device="cuda")
A = [torch.from_numpy(np.ascontiguousarray(rng.standard_normal((R, I)))).cuda().t() for I in dims]
ws = cp.Workspace(dims, R)
nz = cp.norm2(Zd, dims, ws=ws)
out = torch.empty(4, dtype=torch.float64, device="cuda")
for _ in range(n):
    cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws)
    torch.cuda.synchronize()
    print("---- sweep done", flush=True)
