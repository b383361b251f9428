"""cp_fit on a workspace poisoned with 0xFF bytes: which outputs depend on stale workspace."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import cpsynth
import paper_1111_6091_b200 as cp
from gpu_util import dev_factor, dev_tensor

for dims, R in (((40, 36, 30), 6), ((20, 20, 20), 3), ((24, 20, 18, 10), 4), ((64, 64, 64), 16)):
    Z, A0 = cpsynth.random_problem(dims, R, seed=77)
    Zd = dev_tensor(Z)
    Ad = [dev_factor(a) for a in A0]
    res = []
    for fill in (0x00, 0xFF, 0x7F):
        ws = cp.Workspace(dims, R)
        ws.buf.fill_(fill)
        nz = cp.norm2(Zd, dims, ws=ws)
        ws.buf.fill_(fill)
        f, G = cp.fit(Zd, dims, Ad, nz, ws=ws, want_G=True)
        torch.cuda.synchronize()
        res.append((f.cpu().numpy(), [g.cpu().numpy() for g in G]))
    for k in (1, 2):
        df = res[k][0] - res[0][0]
        dG = [float(np.max(np.abs(a - b))) for a, b in zip(res[k][1], res[0][1])]
        print(os.environ.get("TAG", ""), dims, R, hex((0, 0xFF, 0x7F)[k]), "out diff", df, "G diff", dG)
