"""c3 (256^3, R = 8) MTTKRP / sweep device times with L2 flushed before each rep (env knobs apply).
    python tools/c3_knobs.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1111_6091_b200 as cp  # noqa: E402
from paper_1111_6091_b200 import colmajor, empty_factor  # noqa: E402

d3, R3 = (256, 256, 256), 8
Z3 = torch.randn(d3, dtype=torch.float64, device="cuda")
A3 = [colmajor(torch.randn(I, R3, dtype=torch.float64, device="cuda")) for I in d3]
ws = cp.Workspace(d3, R3)
nz = cp.norm2(Z3, d3, ws=ws)
fl = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
M = [empty_factor(I, R3, "cuda") for I in d3]


def flushed(fn, n=30):
    fn()
    tot = 0.0
    for _ in range(n):
        fl.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / n * 1e3


r = [flushed(lambda: cp.mttkrp(Z3, d3, A3, n, M=M[n], ws=ws)) for n in range(3)]
A2 = [a.clone() for a in A3]
A2 = [colmajor(a) for a in A2]
sw = flushed(lambda: cp.als_sweep(Z3, d3, A2, nz, ws=ws))
print(" ".join(f"{x:.1f}" for x in r), f"sweep {sw:.1f} us")
