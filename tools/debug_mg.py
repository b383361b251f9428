import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import cpsynth, oracle
from oracle import mg
import paper_1111_6091_b200 as cp
from gpu_util import dev_factor, dev_tensor, host_factor, relerr
s, R = 20, 2
dims = (s, s, s)
Z = cpsynth.dense_inverse_norm(s)
A0 = cpsynth.uniform_init(dims, R, seed=0)
T0 = [cpsynth.uniform_init(dims, R, seed=10 + t) for t in range(2)]
for cfg in [dict(nu1_setup=0, nu2_setup=0, nuc_setup=0), dict(nu1_setup=1, nu2_setup=0, nuc_setup=0),
            dict(nu1_setup=0, nu2_setup=0, nuc_setup=1), dict(nu1_setup=0, nu2_setup=1, nuc_setup=0), dict()]:
    params = dict(max_setup_cycles=1, max_cycles=1, tol=1e-30, **cfg)
    Zd = dev_tensor(Z); Ad = [dev_factor(a) for a in A0]; Td = [[dev_factor(t) for t in b] for b in T0]
    rep, tr = cp.mg_solve(Zd, dims, Ad, Td, params=cp.MGParams.default(**params))
    Ao, repo, tro = mg.mg_solve(Z, dims, A0, T0, **params)
    print(cfg, [relerr(host_factor(a), b) for a, b in zip(Ad, Ao)], tr[:, 2], tro[:, 2])
