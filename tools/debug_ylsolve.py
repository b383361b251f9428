"""Per-mode error of one sweep vs the oracle on small shapes (debug aid)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import oracle  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402

for dims, R in [((700, 5, 4), 16), ((20, 20, 20), 16), ((64, 64, 64), 16), ((700, 5, 4), 8), ((40, 36, 30), 20), ((20, 20, 20), 3)]:
    Z, A = cpsynth.random_problem(dims, R, seed=100 + R)
    Zd = torch.from_numpy(Z).cuda()
    Ad = [torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t() for a in A]
    nz = cp.norm2(Zd, dims)
    out = cp.als_sweep(Zd, dims, Ad, nz).cpu().numpy()
    Ao, oo = oracle.als_sweep(Z, dims, [a.copy(order="F") for a in A])
    errs = []
    for n in range(3):
        g = Ad[n].cpu().numpy()
        e = np.abs(g - Ao[n]).max(axis=1) / np.abs(Ao[n]).max()
        bad = np.nonzero(e > 1e-9)[0]
        errs.append((n, float(e.max()), bad[:10].tolist(), len(bad)))
    print(dims, R, "status", out[2], out[3], "oracle", oo[2], "f", out[0], oo[0], errs, flush=True)
