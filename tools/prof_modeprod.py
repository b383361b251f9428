"""Time cp_mode_product (restriction Z x_n Phat^T) on a BASELINE config, every mode.
    python tools/prof_modeprod.py [c3] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
_, dims, R, *_ = cpsynth.CONFIGS[name]
Zd = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device="cuda")
P = int(np.prod(dims))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for n in range(len(dims)):
    J = (dims[n] + 1) // 2
    U = torch.randn((dims[n], J), dtype=torch.float64, device="cuda").t()  # J x I col-major
    X, _ = cp.mode_product(Zd, dims, n, U)
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        cp.mode_product(Zd, dims, n, U, X=X)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / reps
    print(f"{name} mode {n}: {ms:.3f} ms  {2.0 * J * P / ms / 1e9:.2f} TFLOP/s")
