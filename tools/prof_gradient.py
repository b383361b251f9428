"""cp_gradient / cp_fit on a BASELINE config a few times (for ncu launch lists).
    python tools/prof_gradient.py [c4a] [reps] [fit|gradient]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4a"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
which = sys.argv[3] if len(sys.argv) > 3 else "gradient"
_, dims, R, *_ = cpsynth.CONFIGS[name]
rng = np.random.default_rng(0)
Zd = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device="cuda")
A = [torch.from_numpy(np.ascontiguousarray(rng.standard_normal((R, I)))).cuda().t() for I in dims]
ws = cp.Workspace(dims, R)
nz = cp.norm2(Zd, dims, ws=ws)
fn = cp.gradient if which == "gradient" else cp.fit
for _ in range(reps):
    fn(Zd, dims, A, nz, ws=ws)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(10):
    fn(Zd, dims, A, nz, ws=ws)
ev[1].record()
torch.cuda.synchronize()
print(f"{name} {which}: {ev[0].elapsed_time(ev[1]) / 10:.4f} ms/call")
