import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
os.environ["CP_SMALL_SWEEP"] = "0"
import numpy as np, torch, cpsynth, oracle
import paper_1111_6091_b200 as cp
from gpu_util import dev_factor, dev_tensor, host_factor, host_tensor, relerr
for dims, R in [((64, 9, 7, 5, 3), 4), ((30, 28, 26, 12), 6), ((20, 9, 7, 5, 3), 3), ((8, 8, 8, 8, 8), 3), ((8, 8, 8, 8, 8, 2), 3)]:
    Z, A = cpsynth.random_problem(dims, R, seed=900 + R)
    nz2 = float(np.vdot(Z, Z))
    Fh = [0.02 * cpsynth.random_matrix(I, R, 40 + k) for k, I in enumerate(dims)]
    Zd = dev_tensor(Z); nzd = cp.norm2(Zd, dims)
    Fd = [dev_factor(f) for f in Fh]
    for ns in (1, 2):
        Ad = [dev_factor(a) for a in A]
        out = host_tensor(cp.als_sweep(Zd, dims, Ad, nzd, F=Fd, nsweeps=ns))
        Ao2 = [a.copy(order="F") for a in A]
        for _ in range(ns): Ao2, oo = oracle.als_sweep(Z, dims, Ao2, F=Fh, normZ2=nz2)
        Ag = [host_factor(a) for a in Ad]
        fa = [float(np.sum(f * a)) for f, a in zip(Fh, Ag)]
        print(dims, R, ns, "f~ gpu", out[1], "oracle", oo[1], "f - sum<F,A> (gpu A)", out[0] - sum(fa), "per-mode <F,A>", fa)
