import sys, os, numpy as np, torch
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root); sys.path.insert(0, os.path.join(root, "tests"))
import cpsynth, oracle
import paper_1111_6091_b200 as cp
from gpu_util import dev_factor, dev_tensor, host_factor, relerr
for dims, R in [((8, 6, 5), 2), ((20, 20, 20), 3), ((16, 12, 10), 4)]:
    Z, A = cpsynth.random_problem(dims, R, seed=1)
    Zd = dev_tensor(Z); Ad = [dev_factor(a) for a in A]
    out = cp.als_sweep(Zd, dims, Ad, cp.norm2(Zd, dims)).cpu().numpy()
    Ao, oo = oracle.als_sweep(Z, dims, A)
    print(dims, R, out, oo, [relerr(host_factor(a), b) for a, b in zip(Ad, Ao)])
    # mode-0 MTTKRP only reference
    M0 = oracle.mttkrp(Z, dims, A, 0)
    print("  M0 norm", np.linalg.norm(M0))
