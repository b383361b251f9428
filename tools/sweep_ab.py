"""cp_als_sweep device time per call (back-to-back, no flush) under environment variants, one
process, same box.  python tools/sweep_ab.py c4b VAR=a,VAR=b ..."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402

name = sys.argv[1]
_, dims, R, *_ = cpsynth.CONFIGS[name]
rng = np.random.default_rng(0)
Zd = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device="cuda")
A0 = [torch.from_numpy(np.ascontiguousarray(rng.standard_normal((R, I)))).cuda().t() for I in dims]
ws = cp.Workspace(dims, R)
nz = cp.norm2(Zd, dims, ws=ws)
out = torch.empty(4, dtype=torch.float64, device="cuda")
for variant in sys.argv[2:] or ["-"]:
    saved = {}
    for kv in variant.split(","):
        if "=" in kv:
            k, v = kv.split("=")
            saved[k] = os.environ.get(k)
            os.environ[k] = v
    A = [a.clone() for a in A0]
    for _ in range(5):
        cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws)
    res = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws)
        e1.record()
        e1.synchronize()
        res.append(e0.elapsed_time(e1) / 50 * 1e3)
    print(f"{name} {variant}: {min(res):.1f} us/sweep (reps {', '.join(f'{x:.1f}' for x in res)})")
    for k, v in saved.items():
        if v is None:
            del os.environ[k]
        else:
            os.environ[k] = v
