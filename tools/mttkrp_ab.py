"""cp_mttkrp device times per mode under environment variants, one process, same box (L2 flushed
before each rep when Z fits in 2x L2, else back-to-back calls).
    python tools/mttkrp_ab.py c3 "CP_MTTKRP_FUSED=0" "CP_MTTKRP_FUSED=1,CP_MTTKRP_FCM=2" ...
(path selectors, include/cp.h; reps via MTTKRP_AB_REPS)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402
from paper_1111_6091_b200 import colmajor, empty_factor  # noqa: E402

name = sys.argv[1]
variants = sys.argv[2:] or ["-"]
reps = int(os.environ.get("MTTKRP_AB_REPS", "30"))
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
        fl.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps * 1e3


ref = None
for v in variants:
    saved = {}
    for kv in v.split(","):
        if "=" in kv:
            k, val = kv.split("=")
            saved[k] = os.environ.get(k)
            os.environ[k] = val
    line = []
    outs = []
    for n in range(len(dims)):
        us = timed(lambda: cp.mttkrp(Z, dims, A, n, M=M[n], ws=ws))
        alg = 8.0 * (P + sum(dims[k] * R for k in range(len(dims)) if k != n) + dims[n] * R)
        line.append(f"m{n} {us:6.1f} us {alg / us / 1e3:5.0f} GB/s {cp.last_launch_count()}L")
        outs.append(M[n].clone())
    if ref is None:
        ref = outs
    d = max(float((a - b).norm() / b.norm()) for a, b in zip(outs, ref))
    print(f"{name} {v:40s} " + " | ".join(line) + f" | rel diff vs first {d:.1e}", flush=True)
    for k, old in saved.items():
        if old is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = old
