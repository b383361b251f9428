"""Small cases of every libcp entry point, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck -- ONE tool per gpurun call, B200_PROFILING.md).
    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py
Covers: the fused small sweep (c0) and the general dimension-tree sweep (c1 shape, tensor-map
stage loads; a 4-way shape: Y_R path), cp_als_sweeps with and without normalization and F, the
odd-I1 scalar path, cp_mttkrp every mode, cp_fit, cp_gradient, both restrictions, the dense mode
product, cp_normalize_sort, cp_als_solve and cp_mg_solve (2 levels)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).cuda().t()


def run(dims, R, seed, F=False, small="1"):
    os.environ["CP_SMALL_SWEEP"] = small
    Z, A = cpsynth.random_problem(dims, R, seed=seed)
    Zd = torch.from_numpy(Z).cuda()
    Ad = [dev(a) for a in A]
    Fd = [dev(0.05 * cpsynth.random_matrix(I, R, 7 + k)) for k, I in enumerate(dims)] if F else None
    ws = cp.Workspace(dims, R)
    nz = cp.norm2(Zd, dims, ws=ws)
    for n in range(len(dims)):
        cp.mttkrp(Zd, dims, Ad, n, ws=ws)
    cp.als_sweep(Zd, dims, Ad, nz, F=Fd, ws=ws)
    cp.als_sweep(Zd, dims, Ad, nz, F=Fd, ws=ws, nsweeps=3)
    cp.als_sweep(Zd, dims, Ad, nz, ws=ws, nsweeps=2, normalize=True)
    cp.fit(Zd, dims, Ad, nz, F=Fd, want_G=True, ws=ws)
    cp.gradient(Zd, dims, Ad, nz, F=Fd, want_G=True, ws=ws)
    cp.normalize_sort(dims, Ad, sort=True, ws=ws)
    torch.cuda.synchronize()


def restrictions(dims, seed):
    Z, _ = cpsynth.random_problem(dims, 1, seed=seed)
    Zd = torch.from_numpy(Z).cuda()
    for n in range(len(dims)):
        wl, wr = cpsynth.transfer_weights(dims[n], seed=seed + n)
        cp.restrict_structured(Zd, dims, n, torch.from_numpy(wl).cuda(), torch.from_numpy(wr).cuda())
        Ic = (dims[n] + 1) // 2
        cp.mode_product(Zd, dims, n, dev(cpsynth.random_matrix(Ic, dims[n], seed + 10 + n)))
    torch.cuda.synchronize()


def solves():
    d = cpsynth.make_config("c0", with_transfer=False)
    dims, R = d["dims"], d["R"]
    Zd = torch.from_numpy(d["Z"]).cuda()
    T0 = [[dev(t) for t in cpsynth.uniform_init(dims, R, seed=10 + t)] for t in range(2)]
    Af = [dev(a) for a in cpsynth.uniform_init((10, 10, 10), R, seed=99)]
    Ad = [dev(a) for a in d["A0"]]
    cp.mg_solve(Zd, dims, Ad, T0, A_fmg=Af, params=cp.MGParams.default(coarsest=10, use_fmg=1, max_cycles=8, tol=1e-9))
    Ad = [dev(a) for a in d["A0"]]
    cp.als_solve(Zd, dims, Ad, tol=1e-9, max_iters=30, check_every=10)
    torch.cuda.synchronize()


if __name__ == "__main__":
    run((20, 20, 20), 3, 1, F=True)            # fused small-sweep kernel (c0 shape)
    run((20, 20, 20), 3, 2, F=True, small="0") # general path, tensor-map stages, PDL chain
    run((50, 48, 46), 8, 3, F=True)            # general path (P > 16384), MMA consumers
    run((9, 8, 7, 6), 5, 4, F=True, small="0") # 4-way: Y_R path
    run((7, 5, 6), 3, 5, small="0")            # odd I1: scalar producer path
    run((130, 9, 6), 20, 6, small="0")         # NT = 3, ragged m-tiles
    restrictions((20, 18, 16), 7)
    solves()
    print("sanitize cases done")
