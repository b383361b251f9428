"""Kernel timeline of one cp_fit (torch.profiler / CUPTI): python tools/trace_fit.py c4a"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4a"
_, dims, R, *_ = cpsynth.CONFIGS[name]
rng = np.random.default_rng(0)
Zd = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device="cuda")
A = [torch.from_numpy(np.ascontiguousarray(rng.standard_normal((R, I)))).cuda().t() for I in dims]
ws = cp.Workspace(dims, R)
nz = cp.norm2(Zd, dims, ws=ws)
for _ in range(3):
    cp.fit(Zd, dims, A, nz, ws=ws)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    cp.fit(Zd, dims, A, nz, ws=ws)
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/trace_fit.json")
ev = sorted([e for e in json.load(open("/tmp/trace_fit.json"))["traceEvents"] if e.get("cat") == "kernel"],
            key=lambda e: e["ts"])
t0 = ev[0]["ts"]
for e in ev:
    print(f"{e['ts'] - t0:9.2f} {e['dur']:8.2f}  {e['name'][:80]}")
