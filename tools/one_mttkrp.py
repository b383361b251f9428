"""One config's cp_mttkrp (mode argv[2]) a few times -- for ncu captures.  CP_MTTKRP_GATHER selects the path."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402
from paper_1111_6091_b200 import colmajor  # noqa: E402

_, dims, R, *_ = cpsynth.CONFIGS[sys.argv[1]]
n = int(sys.argv[2])
Z = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device="cuda")
A = [colmajor(torch.randn(I, R, dtype=torch.float64, device="cuda")) for I in dims]
ws = cp.Workspace(dims, R)
for _ in range(4):
    M = cp.mttkrp(Z, dims, A, n, ws=ws)
torch.cuda.synchronize()
print("ok")
