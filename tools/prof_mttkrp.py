"""Run cp_mttkrp on a BASELINE config, every mode, a few times (for ncu captures).
    python tools/prof_mttkrp.py [c4a] [reps] [modes]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4a"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
modes = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else None
_, dims, R, *_ = cpsynth.CONFIGS[name]
rng = np.random.default_rng(0)
Zd = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device="cuda")
A = [torch.from_numpy(np.ascontiguousarray(rng.standard_normal((R, I)))).cuda().t() for I in dims]
ws = cp.Workspace(dims, R)
modes = modes if modes is not None else list(range(len(dims)))
for _ in range(reps):
    for n in modes:
        cp.mttkrp(Zd, dims, A, n, ws=ws)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for n in modes:
    ev[0].record()
    for _ in range(5):
        cp.mttkrp(Zd, dims, A, n, ws=ws)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 5
    P = int(np.prod(dims))
    print(f"{name} mode {n}: {ms:.3f} ms/call  {8 * P / ms / 1e6:.0f} GB/s (tensor bytes / call time)")
