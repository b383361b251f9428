"""Cycle-by-cycle g traces of the multigrid solve, GPU driver (cp_mg_solve) vs the oracle
(oracle/mg.py), on a BASELINE.json config.  python tools/mg_trace_parity.py c0 10 [fmg] [init]
init: 'u' = U(0,1) test blocks / FMG guess (the paper's P:452), 'n' = N(0,1) (BJ's reading R12)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402
from oracle import mg  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()


def normal_init(dims, R, seed):
    rng = np.random.default_rng(np.random.SeedSequence([cpsynth.SEED_BASE, 5000, seed]))
    return [np.asfortranarray(rng.standard_normal((I, R))) for I in dims]


def main():
    name = sys.argv[1]
    coarsest = int(sys.argv[2])
    fmg = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    init = sys.argv[4] if len(sys.argv) > 4 else "u"
    maxc = int(sys.argv[5]) if len(sys.argv) > 5 else 60
    d = cpsynth.make_config(name, with_transfer=False)
    dims, R, Z, A0 = d["dims"], d["R"], d["Z"], d["A0"]
    mk = cpsynth.uniform_init if init == "u" else normal_init
    T0 = [mk(dims, R, seed=10 + t) for t in range(2)]
    Af = mk(mg.levels(dims, R, coarsest)[-1], R, seed=99)
    kw = dict(coarsest=coarsest, use_fmg=fmg, tol=1e-9, max_cycles=maxc)
    prm = cp.MGParams.default(**kw)
    Ad = [dev(a) for a in A0]
    rep, tr = cp.mg_solve(torch.from_numpy(Z).cuda(), dims, Ad, [[dev(t) for t in b] for b in T0],
                          A_fmg=[dev(a) for a in Af], params=prm)
    t0 = time.time()
    Ao, repo, tro = mg.mg_solve(Z, dims, A0, T0, A_fmg=Af, **kw)
    n = min(len(tr), len(tro))
    rows = [{"cycle": int(tro[k, 1]), "phase": int(tro[k, 0]), "g_oracle": float(tro[k, 2]),
             "g_gpu": float(tr[k, 2]), "rel": float(abs(tr[k, 2] - tro[k, 2]) / abs(tro[k, 2]))} for k in range(n)]
    print(json.dumps({"config": name, "coarsest": coarsest, "fmg": fmg, "init": init,
                      "gpu": {k: rep[k] for k in ("g", "cycles", "setup_cycles", "solve_cycles", "levels", "status",
                                                 "seconds", "fit_seconds")},
                      "oracle": {k: (float(v) if isinstance(v, (float, np.floating)) else v) for k, v in repo.items()},
                      "oracle_seconds": time.time() - t0, "trace": rows}))


if __name__ == "__main__":
    main()
