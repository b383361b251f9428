"""Multigrid vs ALS solve times on a config (GPU).
    python tools/mg_bench.py [c1|dense50] [R|-] [tol] [coarsest]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402


def problem(name, R=None, coarsest=0):
    if name.startswith("dense"):
        s = int(name[5:])
        R = R or 3
        dims = (s, s, s)
        Z = cpsynth.dense_inverse_norm(s)
        A0 = cpsynth.uniform_init(dims, R, seed=0)
        T0 = [cpsynth.uniform_init(dims, R, seed=10 + t) for t in range(2)]
        Af = cpsynth.uniform_init(cp.mg_levels(dims, R, coarsest)[-1], R, seed=99)
        return dims, R, Z, A0, T0, Af
    d = cpsynth.make_config(name, with_transfer=False)
    dims, R = d["dims"], d["R"]
    T0 = [cpsynth.uniform_init(dims, R, seed=10 + t) for t in range(2)]
    Af = cpsynth.uniform_init(cp.mg_levels(dims, R, coarsest)[-1], R, seed=99)
    return dims, R, d["Z"], d["A0"], T0, Af


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()


KEYS = ("g", "cycles", "setup_cycles", "solve_cycles", "levels", "status", "seconds", "fit_seconds")


def run(name, R=None, tol=1e-10, max_als=10000, coarsest=0, max_cycles=500, als=True):
    """ML, ML+FMG (the paper's P:492 combination) and ML+FMG with reading R29's guard, plus the
    plain ALS solve, to g < tol.  seconds include the stopping tests; seconds_excl_stop excludes
    their device time (the paper's timings exclude the stopping criterion)."""
    dims, R, Z, A0, T0, Af = problem(name, R, coarsest)
    Zd = torch.from_numpy(Z).cuda()
    out = {"problem": name, "dims": list(dims), "R": R, "tol": tol, "coarsest": coarsest or 2 * R,
           "levels_sizes": [list(l) for l in cp.mg_levels(dims, R, coarsest)]}
    for key, fmg, guard in (("ml", 0, 0), ("ml_fmg", 1, 0), ("ml_fmg_guard_R29", 1, 1)):
        Ad = [dev(a) for a in A0]
        prm = cp.MGParams.default(use_fmg=fmg, fmg_guard=guard, tol=tol, coarsest=coarsest, max_cycles=max_cycles)
        rep, tr = cp.mg_solve(Zd, dims, Ad, [[dev(t) for t in b] for b in T0], A_fmg=[dev(a) for a in Af], params=prm)
        r = {k: rep[k] for k in KEYS}
        r["seconds_excl_stop"] = rep["seconds"] - rep["fit_seconds"]
        r["outcome"] = "converged" if rep["status"] == 0 else (
            "unsuccessful (cycle limit)" if rep["status"] == 1 else f"failed (status {int(rep['status'])})")
        out[key] = r
    if als:
        Ad = [dev(a) for a in A0]
        out["als"] = cp.als_solve(Zd, dims, Ad, tol=tol, max_iters=max_als, check_every=1)
        # the same ALS with the stopping test every 10 sweeps: the 10 sweeps between tests replay as
        # one CUDA graph (the loop is launch-bound at these sizes)
        Ad = [dev(a) for a in A0]
        out["als_check10_graph"] = cp.als_solve(Zd, dims, Ad, tol=tol, max_iters=max_als, check_every=10)
    return out


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    R = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
    tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-10
    coarsest = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    run(name, R, tol, coarsest=coarsest)  # warm-up (kernel loading, plans)
    print(json.dumps(run(name, R, tol, coarsest=coarsest)))
