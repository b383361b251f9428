"""Diagnose test_chained_calls_without_sync_match_synced: which output of the chain differs."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import cpsynth
import paper_1111_6091_b200 as cp
from gpu_util import dev_factor, dev_tensor, host_factor, host_tensor

dims, R = (40, 36, 30), 6
Z, A0 = cpsynth.random_problem(dims, R, seed=77)
wl, wr = cpsynth.transfer_weights(dims[1], seed=5)
U = np.asfortranarray(cpsynth.random_matrix(12, dims[2], seed=6))
names = ["out", "X1", "X2", "fit", "M", "A0", "A1", "A2"]


def poison():
    if os.environ.get("POISON"):
        t = torch.full((64 << 20,), 0xFF, dtype=torch.uint8, device="cuda")
        del t


def chain(sync, upto=9):
    poison()
    Zd = dev_tensor(Z)
    Ad = [dev_factor(a) for a in A0]
    ws = cp.Workspace(dims, R)
    s = (lambda: torch.cuda.synchronize()) if sync else (lambda: None)
    nz = cp.norm2(Zd, dims, ws=ws); s()
    out = cp.als_sweep(Zd, dims, Ad, nz, ws=ws); s()
    X1, d1 = cp.restrict_structured(Zd, dims, 1, torch.from_numpy(wl).cuda(), torch.from_numpy(wr).cuda()); s()
    X2, d2 = cp.mode_product(X1, d1, 2, dev_factor(U)); s()
    f, _ = cp.fit(Zd, dims, Ad, nz, ws=ws); s()
    M = cp.mttkrp(Zd, dims, Ad, 0, ws=ws); s()
    torch.cuda.synchronize()
    return [host_tensor(t) for t in (out, X1, X2, f, M)] + [host_factor(a) for a in Ad]


ref = chain(True)
for trial in range(3):
    for tag, sync in (("nosync", False), ("sync", True)):
        got = chain(sync)
        bad = [(n, float(np.max(np.abs(a - b)))) for n, a, b in zip(names, got, ref) if not np.array_equal(a, b)]
        print(os.environ.get("CP_PDL", "-"), trial, tag, bad if bad else "identical")
print("ref fit", ref[3])
print("got fit", got[3])
# fit alone on the post-sweep factors, fresh workspace
Zd = dev_tensor(Z)
Ad = [torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t() for a in ref[5:8]]
nz = cp.norm2(Zd, dims)
f, _ = cp.fit(Zd, dims, Ad, nz)
print("fresh fit", f.cpu().numpy())
