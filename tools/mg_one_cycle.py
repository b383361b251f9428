"""The setup cycles + one FAS solve cycle of BASELINE.json c1 (5 levels) -- for ncu launch lists of
the V-cycle.  python tools/mg_one_cycle.py [c1] [coarsest]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()


name = sys.argv[1] if len(sys.argv) > 1 else "c1"
coarsest = int(sys.argv[2]) if len(sys.argv) > 2 else 0
d = cpsynth.make_config(name, with_transfer=False)
dims, R = d["dims"], d["R"]
T0 = [cpsynth.uniform_init(dims, R, seed=10 + t) for t in range(2)]
Zd = torch.from_numpy(d["Z"]).cuda()
prm = cp.MGParams.default(max_cycles=int(os.environ.get("CYC", "6")),
                          tol=1e-30, coarsest=coarsest)
rep, tr = cp.mg_solve(Zd, dims, [dev(a) for a in d["A0"]], [[dev(t) for t in b] for b in T0], params=prm)
torch.cuda.synchronize()
print(rep)
