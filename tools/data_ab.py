"""Does the c4a sweep time depend on the data or on where the tensor was allocated?  The same
sweep loop (one cp_als_sweeps(50) call, CUDA events, per-launch profile) on
  a) device randn Z + randn factors (tools/time_sweep.py),
  b) the cpsynth c4a tensor and initial factors (bench.py),
  c) the cpsynth tensor copied into a fresh device allocation,
  d) the randn tensor with the cpsynth factors.
    python tools/data_ab.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402

dims, R = (512, 512, 512), 16
rng = np.random.default_rng(0)
Zr = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device="cuda")
Ar = [torch.from_numpy(np.ascontiguousarray(rng.standard_normal((R, I)))).cuda().t() for I in dims]
d = cpsynth.make_config("c4a", with_transfer=False)
Zc = torch.from_numpy(d["Z"]).cuda()
Ac = [torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t() for a in d["A0"]]
Zc2 = torch.empty_like(Zr)
Zc2.copy_(Zc)
ws = cp.Workspace(dims, R)
out = torch.empty(4, dtype=torch.float64, device="cuda")


def run(label, Z, A0):
    nz = cp.norm2(Z, dims, ws=ws)
    for rep in range(2):
        A = [a.clone() for a in A0]
        cp.als_sweep(Z, dims, A, nz, out=out, ws=ws, nsweeps=10)
        torch.cuda.synchronize()
        res = []
        for prof in (False, True):
            cp.profile_enable(prof)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(4):
                cp.als_sweep(Z, dims, A, nz, out=out, ws=ws, nsweeps=50)
            e1.record()
            torch.cuda.synchronize()
            n, pms, pb = cp.profile_read()
            cp.profile_enable(False)
            res.append((e0.elapsed_time(e1) / 200, pms / max(1, n)))
        print(f"{label:28s} sweep {res[0][0]:.4f} ms (profiled {res[1][0]:.4f}); stream launch {res[1][1] * 1e3:.1f} us; "
              f"status {out[2].item()} f {out[0].item():.4e}", flush=True)


run("a) randn Z, randn A", Zr, Ar)
run("b) cpsynth Z, cpsynth A0", Zc, Ac)
run("c) cpsynth Z (copy), cpsynth A0", Zc2, Ac)
run("d) randn Z, cpsynth A0", Zr, Ac)
run("e) cpsynth Z, randn A", Zc, Ar)
