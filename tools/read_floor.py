"""Cold single-pass floor at one config: device time of one call after an L2 flush that leaves the
cache cold AND clean (256 MiB write, then a 256 MiB read of another buffer), for a plain
streaming read of Z (torch sum, cp_norm2) against cp_mttkrp of every mode and one sweep; graph
replays (no host time inside the events).   python tools/read_floor.py c3"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402
from paper_1111_6091_b200 import colmajor, empty_factor  # noqa: E402

name = sys.argv[1]
_, dims, R, *_ = cpsynth.CONFIGS[name]
Z = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device="cuda")
A = [colmajor(torch.randn(I, R, dtype=torch.float64, device="cuda")) for I in dims]
ws = cp.Workspace(dims, R)
Ms = [empty_factor(I, R, "cuda") for I in dims]
nz = cp.norm2(Z, dims, ws=ws)
out = torch.empty(4, dtype=torch.float64, device="cuda")
red = torch.empty((), dtype=torch.float64, device="cuda")
fl = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
fl2 = torch.ones(256 * 2**17, dtype=torch.float64, device="cuda")
cur = lambda: torch.cuda.current_stream()  # noqa: E731
ops = {
    "torch.sum(Z)": lambda: torch.sum(Z.view(-1), 0, out=red),
    "cp_norm2": lambda: cp.norm2(Z, dims, out=nz, ws=ws, stream=cur()),
}
for n in range(len(dims)):
    ops[f"cp_mttkrp m{n}"] = (lambda n=n: cp.mttkrp(Z, dims, A, n, M=Ms[n], ws=ws, stream=cur()))
ops["cp_als_sweep"] = lambda: cp.als_sweep(Z, dims, A, nz, out=out, ws=ws, stream=cur())
P = int(np.prod(dims))
for label, fn in ops.items():
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for _ in range(20):
        fl.zero_()
        fl2.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    us = float(np.median(ts))
    print(f"{name} {label:16s} clean-cold {us:7.1f} us  = {8.0 * P / us / 1e3:6.0f} GB/s of Z", flush=True)
