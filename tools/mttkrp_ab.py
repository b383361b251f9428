"""cp_mttkrp device times per mode (L2 flushed before each rep), gather path vs prep path
(CP_MTTKRP_FCM=1/0).  python tools/mttkrp_ab.py c3 [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402
from paper_1111_6091_b200 import colmajor, empty_factor  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
_, dims, R, *_ = cpsynth.CONFIGS[name]
P = int(np.prod(dims))
Z = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device="cuda")
A = [colmajor(torch.randn(I, R, dtype=torch.float64, device="cuda")) for I in dims]
ws = cp.Workspace(dims, R)
M = [empty_factor(I, R, "cuda") for I in dims]
fl = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
flush = 8 * P <= 2 * 126 * 2**20


def timed(fn):
    fn()
    if not flush:  # back-to-back calls between two events (the bench rows' timing)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3
    tot = 0.0
    for _ in range(reps):
        if flush:
            fl.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps * 1e3


res = {}
for g in ("1", "0"):
    os.environ["CP_MTTKRP_FCM"] = g
    for n in range(len(dims)):
        us = timed(lambda: cp.mttkrp(Z, dims, A, n, M=M[n], ws=ws))
        alg = 8.0 * (P + sum(dims[k] * R for k in range(len(dims)) if k != n) + dims[n] * R)
        res[(g, n)] = (us, alg / us / 1e3, cp.last_launch_count())
for n in range(len(dims)):
    print(f"{name} mode {n}: fcm {res[('1', n)][0]:.1f} us ({res[('1', n)][1]:.0f} GB/s, {res[('1', n)][2]} launches)"
          f" | prep {res[('0', n)][0]:.1f} us ({res[('0', n)][1]:.0f} GB/s, {res[('0', n)][2]} launches)")
os.environ["CP_MTTKRP_FCM"] = "1"
Mg = [cp.mttkrp(Z, dims, A, n).clone() for n in range(len(dims))]
os.environ["CP_MTTKRP_FCM"] = "0"
Mp = [cp.mttkrp(Z, dims, A, n).clone() for n in range(len(dims))]
print("max rel diff fcm vs prep:", max(float((a - b).norm() / b.norm()) for a, b in zip(Mg, Mp)))
