"""Kernel timeline of a few sweeps via torch.profiler (CUPTI activity records; no replay, no
serialisation): python tools/trace_sweep.py c4a [sweeps] -> prints per-kernel start/end offsets."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402

name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
_, dims, R, *_ = cpsynth.CONFIGS[name]
rng = np.random.default_rng(0)
Zd = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device="cuda")
A = [torch.from_numpy(np.ascontiguousarray(rng.standard_normal((R, I)))).cuda().t() for I in dims]
ws = cp.Workspace(dims, R)
nz = cp.norm2(Zd, dims, ws=ws)
out = torch.empty(4, dtype=torch.float64, device="cuda")
for _ in range(10):
    cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(n):
        cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws)
    torch.cuda.synchronize()
path = f"/tmp/trace_{name}.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
prev_end = None
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("CP_"))
print(f"# {name} {tag}")
for e in ev:
    s, d = e["ts"] - t0, e["dur"]
    gap = (s - prev_end) if prev_end is not None else 0.0
    print(f"{s:9.2f} {d:8.2f} gap {gap:7.2f}  {e['name'][:70]}")
    prev_end = s + d
