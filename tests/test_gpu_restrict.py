"""GPU parity of cp_restrict_structured against the oracle's dense definition
(oracle.mg.restrict_structured: P from the weights, Phat = P L^{-T}, dense mode product):
ragged shapes for every mode (odd / even / 1 / 2 sizes, N = 1..5), the c3 config in full, and
sampled fibers of the c4a tensor at full size.  Tolerance: 1e-12 relative (BASELINE.json,
mode-product outputs)."""
import numpy as np
import pytest
import torch

import cpsynth
from oracle import mg
from gpu_util import relerr

import paper_1111_6091_b200 as cp

pytestmark = pytest.mark.gpu

SHAPES = [((9, 6, 5), 0), ((9, 6, 5), 1), ((9, 6, 5), 2), ((8, 7, 4), 0), ((2, 3, 4), 0), ((1, 5, 3), 0),
          ((5, 2, 7), 1), ((3, 4, 1), 2), ((64, 9, 7, 5, 3), 0), ((64, 9, 7, 5, 3), 3), ((1031,), 0),
          ((70, 33), 0), ((70, 33), 1), ((40, 36, 30), 1), ((130, 3, 3), 0), ((3, 3, 130), 2)]


def run(Z, dims, mode, wl, wr):
    Zd = torch.from_numpy(np.ascontiguousarray(Z)).cuda()
    X, nd = cp.restrict_structured(Zd, dims, mode, torch.from_numpy(wl).cuda(), torch.from_numpy(wr).cuda())
    return X.cpu().numpy(), nd


@pytest.mark.parametrize("dims,mode", SHAPES)
def test_restrict_structured_ragged(dims, mode):
    Z, _ = cpsynth.random_problem(dims, 1, seed=40 + mode + len(dims))
    wl, wr = cpsynth.transfer_weights(dims[mode], seed=dims[mode])
    Xg, nd = run(Z, dims, mode, wl, wr)
    Xo, ndo = mg.restrict_structured(Z, dims, mode, wl, wr)
    assert list(nd) == list(ndo)
    assert relerr(Xg.reshape(-1), Xo.reshape(-1)) <= 1e-12


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_restrict_structured_c3_full(mode):
    d = cpsynth.make_config("c3", with_transfer=False)
    dims, Z = d["dims"], d["Z"]
    wl, wr = cpsynth.transfer_weights(dims[mode], seed=256 + mode)
    Xg, _ = run(Z, dims, mode, wl, wr)
    Xo, _ = mg.restrict_structured(Z, dims, mode, wl, wr)
    assert relerr(Xg.reshape(-1), Xo.reshape(-1)) <= 1e-12


def test_restrict_structured_c4a_sampled_fibers():
    """Full-size c4a (512^3), the launch configuration bench.py times: 64 sampled output fibers
    per mode against Phat^T applied to the same input fibers on the host."""
    d = cpsynth.make_config("c4a", with_transfer=False)
    dims, Z = d["dims"], d["Z"]
    Zt = Z.reshape(tuple(reversed(dims)))          # index [i3, i2, i1]
    Zd = torch.from_numpy(Z).cuda()
    rng = np.random.default_rng(5)
    for mode in range(3):
        wl, wr = cpsynth.transfer_weights(dims[mode], seed=512 + mode)
        X, nd = cp.restrict_structured(Zd, dims, mode, torch.from_numpy(wl).cuda(), torch.from_numpy(wr).cuda())
        Xt = X.cpu().numpy().reshape(tuple(reversed(nd)))
        Ph = mg.transfer(mg.interpolation_from_weights(dims[mode], wl, wr))
        ax = 2 - mode                              # numpy axis of this mode
        for _ in range(64):
            idx = [int(rng.integers(0, n)) for n in reversed(dims)]
            sl = tuple(slice(None) if a == ax else idx[a] for a in range(3))
            assert relerr(Xt[sl], Ph.T @ Zt[sl]) <= 1e-12
        del X


def test_restrict_matches_dense_mode_product_on_gpu():
    """Same result as cp_mode_product with the dense Phat^T (up to rounding)."""
    dims, mode = (40, 36, 30), 1
    Z, _ = cpsynth.random_problem(dims, 1, seed=9)
    wl, wr = cpsynth.transfer_weights(dims[mode], seed=3)
    Ph = mg.transfer(mg.interpolation_from_weights(dims[mode], wl, wr))
    Zd = torch.from_numpy(Z).cuda()
    U = cp.colmajor(torch.from_numpy(np.ascontiguousarray(Ph.T)).cuda())
    Xd, _ = cp.mode_product(Zd, dims, mode, U)
    Xs, _ = cp.restrict_structured(Zd, dims, mode, torch.from_numpy(wl).cuda(), torch.from_numpy(wr).cuda())
    assert relerr(Xs.cpu().numpy(), Xd.cpu().numpy()) <= 1e-12


def test_restrict_rejects_bad_arguments():
    Zd = torch.zeros(4, 4, dtype=torch.float64, device="cuda")
    w = torch.zeros(4, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        cp.restrict_structured(Zd, (4, 4), 0, w[:3], w)
    L = cp.lib()
    import ctypes
    d = (ctypes.c_int64 * 2)(4, 4)
    assert L.cp_restrict_structured(2, d, ctypes.c_void_p(Zd.data_ptr()), 2, ctypes.c_void_p(w.data_ptr()),
                                    ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(Zd.data_ptr()),
                                    ctypes.c_void_p(w.data_ptr()), 32, None) == cp.CP_EINVAL


def test_restrict_chained_galerkin_all_modes():
    """The multigrid driver's Galerkin tensor: restrictions of every mode chained on the stream
    with no host synchronization in between (each call reads the previous call's output)."""
    dims = (66, 40, 34)
    Z, _ = cpsynth.random_problem(dims, 1, seed=13)
    W = [cpsynth.transfer_weights(I, seed=70 + n) for n, I in enumerate(dims)]
    Xd = torch.from_numpy(Z).cuda()
    cur = list(dims)
    for n in range(3):
        Xd, cur = cp.restrict_structured(Xd, cur, n, torch.from_numpy(W[n][0]).cuda(), torch.from_numpy(W[n][1]).cuda())
    Xo, curo = Z, list(dims)
    for n in range(3):
        Xo, curo = mg.restrict_structured(Xo, curo, n, *W[n])
    assert list(cur) == list(curo)
    assert relerr(Xd.cpu().numpy().reshape(-1), Xo.reshape(-1)) <= 1e-12
