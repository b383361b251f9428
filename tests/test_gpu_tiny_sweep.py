"""The single-warp sweep kernel for the tiniest multigrid levels (tiny_sweep.cu: N <= 4, R <= 4,
every mode with at most 32 columns; the coarsest-level relaxation of the V-cycle, Table 1
nu_c = 50): nu sweeps in one launch against nu oracle sweeps (P:121,
eq:relaxinnersolve P:356-358) with and without the FAS right-hand side, the setup-phase variant
with eq:ALSnorm after every sweep, the CP_ENOTSPD report -- and factors BITWISE equal
to the 512-thread fused kernel it replaces (CP_TINY_SWEEP=0): the multigrid solves are sensitive
to rounding-level changes on their coarsest level (DESIGN reading R31), so the kernel keeps every
expression and summation order of small_sweep_kernel."""
import math

import numpy as np
import pytest

import cpsynth
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1111_6091_b200 as cp  # noqa: E402
from gpu_util import dev_factor, dev_tensor, host_factor, host_tensor, relerr  # noqa: E402

SHAPES = [
    ((4, 4, 4), 3),          # c1 / dense-problem coarsest level: 16 columns per mode
    ((5, 5, 5), 3),          # 25 columns: 32-lane tree with 7 empty lanes
    ((5, 4, 3), 2),
    ((4, 4, 4), 1),
    ((6, 5, 4), 4),          # R = 4; 20 / 24 / 30 columns
    ((2, 3, 2, 3), 3),       # N = 4
    ((16, 2, 2), 2),         # 32 columns in modes 1, 2
    ((6, 5), 2),             # N = 2
    ((4, 1, 5), 1),          # degenerate mode
    ((7, 7, 7), 3),          # 49 columns: not eligible -> the 512-thread kernel (same results)
]


def _run(Z, dims, A, F, nu, tiny, monkeypatch, normalize=False):
    monkeypatch.setenv("CP_SMALL_SWEEP", "1")
    monkeypatch.setenv("CP_TINY_SWEEP", tiny)
    Zd, Ad = dev_tensor(Z), [dev_factor(a) for a in A]
    Fd = None if F is None else [dev_factor(f) if f is not None else None for f in F]
    out = host_tensor(cp.als_sweep(Zd, dims, Ad, cp.norm2(Zd, dims), F=Fd, nsweeps=nu, normalize=normalize))
    assert cp.last_launch_count() == 1
    return [host_factor(a) for a in Ad], out


def _check(Ag, og, Ao, oo, nz2, tol=1e-10):
    assert og[2] == 0 == oo[2]
    for a, b in zip(Ag, Ao):
        assert relerr(a, b) <= tol
    assert abs(og[0] - oo[0]) <= tol * abs(oo[0]) + 1e-14 * 0.5 * nz2
    assert abs(og[1] - oo[1]) <= tol * abs(oo[1]) + 1e-14 * 0.5 * nz2


@pytest.mark.parametrize("nu", [1, 6])
@pytest.mark.parametrize("with_F", [False, True])
@pytest.mark.parametrize("dims,R", SHAPES)
def test_tiny_sweeps_vs_oracle(dims, R, with_F, nu, monkeypatch):
    Z, A = cpsynth.random_problem(dims, R, seed=60 + R)
    N = len(dims)
    if not all(R <= int(np.prod(dims)) // d for d in dims):
        pytest.skip("Gamma singular for every iterate")
    F = [0.05 * cpsynth.random_matrix(dims[k], R, 7 + k) if k != 1 else None for k in range(N)] if with_F else None
    nz2 = float(np.vdot(Z, Z))
    Ag, og = _run(Z, dims, A, F, nu, "1", monkeypatch)
    Ao = [a.copy(order="F") for a in A]
    for _ in range(nu):
        Ao, oo = oracle.als_sweep(Z, dims, Ao, F=F, normZ2=nz2)
    _check(Ag, og, Ao, oo, nz2)
    # the 512-thread fused kernel from the same state: bitwise the same factors; f, f~ summed over
    # lanes instead of threads (rounding level)
    As, os_ = _run(Z, dims, A, F, nu, "0", monkeypatch)
    for a, b in zip(Ag, As):
        assert np.array_equal(a.view(np.int64), b.view(np.int64))
    assert abs(og[0] - os_[0]) <= 1e-13 * abs(os_[0]) + 1e-15 * nz2
    assert abs(og[1] - os_[1]) <= 1e-13 * abs(os_[1]) + 1e-15 * nz2


@pytest.mark.parametrize("dims,R", [((4, 4, 4), 3), ((5, 5, 5), 3), ((6, 5, 4), 4), ((2, 3, 2, 3), 2)])
def test_tiny_sweeps_normalized_vs_oracle(dims, R, monkeypatch):
    Z, A = cpsynth.random_problem(dims, R, seed=70 + R)
    nz2 = float(np.vdot(Z, Z))
    nu = 5
    Ag, og = _run(Z, dims, A, None, nu, "1", monkeypatch, normalize=True)
    Ao = [a.copy(order="F") for a in A]
    for _ in range(nu):
        Ao, oo = oracle.als_sweep(Z, dims, Ao, normZ2=nz2)
        Ao, _ = oracle.normalize_sort(dims, Ao, sort=False)
    _check(Ag, og, Ao, oo, nz2)
    As, _ = _run(Z, dims, A, None, nu, "0", monkeypatch, normalize=True)
    for a, b in zip(Ag, As):
        assert np.array_equal(a.view(np.int64), b.view(np.int64))


def test_tiny_fifty_coarsest_sweeps_c1_level(monkeypatch):
    """nu_c = 50 sweeps on a 4^3 level (Table 1): the trajectory stays within 1e-10 of the oracle."""
    dims, R = (4, 4, 4), 3
    Z, A = cpsynth.random_problem(dims, R, seed=1)
    F = [0.01 * cpsynth.random_matrix(4, R, 3 + k) for k in range(3)]
    nz2 = float(np.vdot(Z, Z))
    Ag, og = _run(Z, dims, A, F, 50, "1", monkeypatch)
    Ao = [a.copy(order="F") for a in A]
    for _ in range(50):
        Ao, oo = oracle.als_sweep(Z, dims, Ao, F=F, normZ2=nz2)
    _check(Ag, og, Ao, oo, nz2, tol=1e-9)


@pytest.mark.parametrize("R,col", [(2, 0), (4, 3)])
def test_tiny_singular_gamma_reports_enotspd(R, col, monkeypatch):
    dims = (6, 5, 4)
    Z, A = cpsynth.random_problem(dims, R, seed=9)
    A[1][:, col] = 0.0
    Ag, og = _run(Z, dims, A, None, 3, "1", monkeypatch)
    _, oo = oracle.als_sweep(Z, dims, A)
    assert og[2] == cp.CP_ENOTSPD == oo[2]
    assert og[3] == oo[3] == 0
    assert math.isnan(og[0]) and math.isnan(og[1])


def test_tiny_deterministic(monkeypatch):
    dims, R = (5, 5, 5), 3
    Z, A = cpsynth.random_problem(dims, R, seed=4)
    ref = _run(Z, dims, A, None, 9, "1", monkeypatch)
    for _ in range(3):
        got = _run(Z, dims, A, None, 9, "1", monkeypatch)
        for a, b in zip(ref[0], got[0]):
            assert np.array_equal(a.view(np.int64), b.view(np.int64))
        assert np.array_equal(ref[1].view(np.int64), got[1].view(np.int64))
