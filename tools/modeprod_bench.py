"""Dense mode product (cp_mode_product, DMMA GEMM) timing: c4a / c3 restriction with Phat^T, every mode."""
import sys
import torch
import numpy as np
sys.path.insert(0, '.')
import paper_1111_6091_b200 as cp
for dims, J in [((512, 512, 512), 256), ((256, 256, 256), 128)]:
    Z = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device='cuda')
    for n in range(3):
        U = cp.colmajor(torch.randn(J, dims[n], dtype=torch.float64, device='cuda'))
        nd = list(dims); nd[n] = J
        X = torch.empty(tuple(reversed(nd)), dtype=torch.float64, device='cuda')
        for _ in range(2): cp.mode_product(Z, dims, n, U, X=X)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): cp.mode_product(Z, dims, n, U, X=X)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(dims, "mode", n, f"{ms:.3f} ms", f"{2.0 * J * np.prod(dims) / ms / 1e9:.1f} TFLOP/s")
