"""Time cp_als_sweep (device, CUDA events) on a config with random data:
    python tools/time_sweep.py c4a [reps]
Prints ms/sweep and the streaming kernels' live average (cp_profile_*)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
nsw = int(os.environ.get("NSW", "1"))  # sweeps per call (cp_als_sweeps steady state when > 1)
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
cp.profile_enable(os.environ.get("NOPROF", "0") != "1")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
import time
e0.record()
th = time.perf_counter()
for _ in range(max(1, reps // nsw)):
    cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws, nsweeps=nsw)
reps = max(1, reps // nsw) * nsw
th = (time.perf_counter() - th) / reps * 1e3
e1.record()
torch.cuda.synchronize()
n, pms, pb = cp.profile_read()
cp.profile_enable(False)
ms = e0.elapsed_time(e1) / reps
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("CP_"))
gbs = pb / max(1, n) / (pms / max(1, n)) / 1e6 if pms > 0 else float("nan")
print(f"{name} {tag}: {ms:.4f} ms/sweep; stream kernels {pms / max(1, n):.4f} ms avg, "
      f"{gbs:.0f} GB/s alg, share {pms / reps / ms:.3f}; "
      f"status {out[2].item()}; host {th:.4f} ms/call", flush=True)
if os.environ.get("GRAPH", "0") == "1":
    cp.profile_enable(False)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(10):
                cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps // 10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"  graph: {e0.elapsed_time(e1) / (reps // 10 * 10):.4f} ms/sweep; status {out[2].item()}", flush=True)
