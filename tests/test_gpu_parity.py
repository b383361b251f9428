"""GPU parity: libcp.so (through the Python binding over the C ABI) against the CPU oracle on
identical seeded inputs.  Tolerances (BASELINE.json north star):
  MTTKRP and mode products: relative Frobenius error <= 1e-12 per output array;
  factors and f after each sweep: <= 1e-10 relative (f: 1e-10*f + 1e-14*||Z||^2/2);
  g: 1e-10*g + 1e-13.
"""
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

RAGGED = [
    ((3, 4, 2), 2),
    ((5, 7, 3), 3),          # odd I1: scalar fallback path
    ((2, 3, 2, 3), 3),
    ((20, 20, 20), 3),
    ((6, 1, 5), 1),
    ((1, 4, 3), 2),
    ((33, 2), 5),            # N = 2
    ((64, 9, 7, 5, 3), 4),   # N = 5
    ((1030, 3, 2), 7),       # I1 > 512: row blocks
    ((1031, 2, 3), 2),       # odd and > 256: scalar row blocks
    ((700, 5, 4), 16),       # mode-0 narrow row blocks
    ((8, 8, 8), 32),         # R = CP_MAX_R
    ((512, 3, 4), 16),
    ((96, 5, 6, 7), 10),
    ((2, 2, 2, 2, 2, 2, 2, 2), 3),  # N = CP_MAX_N
]
# shapes that exercise the tensor-core consumer geometry (stream_mma.cuh): NT = 3, 4 n-tiles with
# masked ranks, ragged m-tiles, two row blocks with a ragged last block, k-split groups
MMA_SHAPES = [
    ((130, 9, 6), 20),       # NT = 3, 17 m-tiles over 8 warps x MT 3
    ((258, 7, 5), 25),       # NT = 4, two row blocks (136 + 122 rows)
    ((40, 36, 30), 20),      # k-split: KS = 4 groups of 2 warps
    ((96, 10, 12), 24),      # NT = 3, KS = 2
]
RAGGED = RAGGED + MMA_SHAPES

_cfg_cache = {}


def config(name):
    if name not in _cfg_cache:
        _cfg_cache.clear()  # keep at most one config (c4a is 1 GiB) in host memory
        _cfg_cache[name] = cpsynth.make_config(name)
    return _cfg_cache[name]


def dev_problem(Z, A):
    return dev_tensor(Z), [dev_factor(a) for a in A]


# ------------------------------------------------------------------------------- ||Z||^2
@pytest.mark.parametrize("dims", [(3,), (7, 5), (20, 20, 20), (5, 7, 3), (1,)])
def test_norm2(dims):
    Z, _ = cpsynth.random_problem(dims, 1, seed=len(dims))
    out = cp.norm2(dev_tensor(Z), dims)
    assert relerr(host_tensor(out)[0], oracle.norm2(Z)) <= 1e-13


# ------------------------------------------------------------------------------- MTTKRP
@pytest.mark.parametrize("dims,R", RAGGED)
def test_mttkrp_ragged(dims, R):
    Z, A = cpsynth.random_problem(dims, R, seed=7 * len(dims) + R)
    Zd, Ad = dev_problem(Z, A)
    for n in range(len(dims)):
        M = host_factor(cp.mttkrp(Zd, dims, Ad, n))
        Mo = oracle.mttkrp(Z, dims, A, n)
        assert relerr(M, Mo) <= 1e-12, (dims, R, n)


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3"])
def test_mttkrp_configs_full(name):
    d = config(name)
    dims, Z, A = d["dims"], d["Z"], d["A0"]
    Zd, Ad = dev_problem(Z, A)
    for n in range(len(dims)):
        M = host_factor(cp.mttkrp(Zd, dims, Ad, n))
        assert relerr(M, oracle.mttkrp(Z, dims, A, n)) <= 1e-12, (name, n)


@pytest.mark.parametrize("name", ["c4a", "c4b"])
def test_mttkrp_configs_sampled_rows(name):
    """Full-size configs at the bench launch configuration: sampled output rows against the
    oracle computed row by row, plus the Kruskal closed form of the noiseless part."""
    d = config(name)
    dims, Z, A = d["dims"], d["Z"], d["A0"]
    Zd, Ad = dev_problem(Z, A)
    rng = np.random.default_rng(3)
    for n in range(len(dims)):
        M = host_factor(cp.mttkrp(Zd, dims, Ad, n))
        rows = sorted(set([0, dims[n] - 1] + list(rng.integers(0, dims[n], 4))))
        for i in rows:
            Mo = oracle.mttkrp(Z, dims, A, n, rows=(i, i + 1))
            assert relerr(M[i], Mo[i]) <= 1e-12, (name, n, i)
    del Zd


def test_mttkrp_kruskal_closed_form_c4a():
    """MTTKRP of the noiseless c4a target T = [[A*]] at full size equals
    A*^(n) (*_{k != n} A*^(k)^T A^(k)) (eq:propKKR) -- a property at any size."""
    _, dims, R, C, *_ = cpsynth.CONFIGS["c4a"]
    rng = np.random.default_rng(11)
    At = cpsynth.congruence_factors(rng, dims, R, C)
    A = [np.asfortranarray(rng.standard_normal((I, R))) for I in dims]
    T = cpsynth.kruskal(At)
    Td = dev_tensor(T)
    del T
    Ad = [dev_factor(a) for a in A]
    for n in range(3):
        H = np.ones((R, R))
        for k in range(3):
            if k != n:
                H *= At[k].T @ A[k]
        M = host_factor(cp.mttkrp(Td, dims, Ad, n))
        assert relerr(M, At[n] @ H) <= 1e-12


# ------------------------------------------------------------------------------- sweep
def _sweep_pair(Z, dims, A, F=None, nsweeps=1, nz2=None):
    """Run nsweeps on both sides from the same A; yield (k, gpu A, gpu out, oracle A, oracle out)."""
    nz2 = float(np.vdot(Z, Z)) if nz2 is None else nz2
    Zd, Ad = dev_problem(Z, A)
    nzd = cp.norm2(Zd, dims)
    Fd = None if F is None else [dev_factor(f) if f is not None else None for f in F]
    Ao = [a.copy(order="F") for a in A]
    ws = cp.Workspace(dims, A[0].shape[1])
    for k in range(nsweeps):
        out = host_tensor(cp.als_sweep(Zd, dims, Ad, nzd, F=Fd, ws=ws))
        Ao, oo = oracle.als_sweep(Z, dims, Ao, F=F, normZ2=nz2)
        yield k, [host_factor(a) for a in Ad], out, Ao, oo


def _check_sweep(Ag, og, Ao, oo, nz2, tol=1e-10):
    if oo[2] != 0:  # singular Gamma (e.g. R > rank possible): both sides must report it
        assert og[2] == oo[2] and og[3] == oo[3]
        return
    assert og[2] == 0
    for a, b in zip(Ag, Ao):
        assert relerr(a, b) <= tol
    assert abs(og[0] - oo[0]) <= tol * abs(oo[0]) + 1e-14 * 0.5 * nz2
    assert abs(og[1] - oo[1]) <= tol * abs(oo[1]) + 1e-14 * 0.5 * nz2


def _well_posed(dims, R):
    """Gamma^(n) can be nonsingular only if Phi^(n) has full column rank: R <= prod_{k!=n} I_k."""
    P = int(np.prod(dims))
    return all(R <= P // d for d in dims)


@pytest.fixture(params=["fused_small", "general"])
def sweep_path(request, monkeypatch):
    """cp_als_sweep runs tensors with P <= 16384 through the fused shared-memory kernel
    (small_sweep.cu); CP_SMALL_SWEEP=0 forces the general multi-kernel path."""
    monkeypatch.setenv("CP_SMALL_SWEEP", "1" if request.param == "fused_small" else "0")
    return request.param


@pytest.mark.parametrize("dims,R", [r for r in RAGGED if r[1] <= 16 and len(r[0]) <= 5 and _well_posed(*r)])
def test_sweep_single_step_ragged(dims, R, sweep_path):
    Z, A = cpsynth.random_problem(dims, R, seed=100 + R)
    nz2 = float(np.vdot(Z, Z))
    for _, Ag, og, Ao, oo in _sweep_pair(Z, dims, A, nsweeps=2, nz2=nz2):
        _check_sweep(Ag, og, Ao, oo, nz2)


@pytest.mark.parametrize("dims,R", [r for r in MMA_SHAPES if _well_posed(*r)])
def test_sweep_single_step_mma_shapes(dims, R):
    Z, A = cpsynth.random_problem(dims, R, seed=300 + R)
    nz2 = float(np.vdot(Z, Z))
    for _, Ag, og, Ao, oo in _sweep_pair(Z, dims, A, nsweeps=2, nz2=nz2):
        _check_sweep(Ag, og, Ao, oo, nz2)


@pytest.mark.parametrize("name,nsweeps", [("c0", 20), ("c1", 20), ("c2", 20), ("c3", 20)])
def test_sweep_trajectory_configs(name, nsweeps):
    """SURVEY 8(c) trajectory protocol: both sides from A0, compared after every sweep (1e-10)."""
    d = config(name)
    dims, Z = d["dims"], d["Z"]
    nz2 = float(np.vdot(Z, Z))
    for k, Ag, og, Ao, oo in _sweep_pair(Z, dims, d["A0"], nsweeps=nsweeps, nz2=nz2):
        _check_sweep(Ag, og, Ao, oo, nz2)


@pytest.mark.parametrize("name", ["c4a", "c4b"])
def test_sweep_full_size_trajectory(name):
    """3 sweeps at the full sizes (the bench launch configuration), every factor and
    f compared with the oracle after every sweep."""
    d = config(name)
    dims, Z = d["dims"], d["Z"]
    nz2 = float(np.vdot(Z, Z))
    for k, Ag, og, Ao, oo in _sweep_pair(Z, dims, d["A0"], nsweeps=3, nz2=nz2):
        _check_sweep(Ag, og, Ao, oo, nz2)


@pytest.mark.parametrize("dims,R", [((12, 10, 9), 3), ((64, 9, 7, 5, 3), 4), ((96, 10, 12), 24)])
def test_sweep_with_rhs(sweep_path, dims, R):
    """BNGS with a FAS right-hand side (eq:relaxinnersolve), including NULL entries; f and f~.
    (64, 9, 7, 5, 3): the mode-0 ylsolve runs 2 clusters while every other blocking of the shape
    has 1 -- the per-cluster <F, A> and Gram partials need their own slots (a round-1 layout bug
    counted one cluster's <F, A> into mode 1's)."""
    Z, A = cpsynth.random_problem(dims, R, seed=5)
    F = [0.05 * cpsynth.random_matrix(dims[k], R, 1 + k) if k != 1 else None for k in range(len(dims))]
    nz2 = float(np.vdot(Z, Z))
    for _, Ag, og, Ao, oo in _sweep_pair(Z, dims, A, F=F, nsweeps=3, nz2=nz2):
        _check_sweep(Ag, og, Ao, oo, nz2)


@pytest.mark.parametrize("R,col", [(2, 0), (8, 5)])
def test_sweep_singular_gamma_reports_enotspd(sweep_path, R, col):
    """A zero factor column makes Gamma^(0) singular (Keller condition P:362); R = 8 runs the
    fused kernel's warp Cholesky and fails at pivot j = col, mid-factorization."""
    dims = (6, 5, 4)
    Z, A = cpsynth.random_problem(dims, R, seed=9)
    A[1][:, col] = 0.0
    Zd, Ad = dev_problem(Z, A)
    out = host_tensor(cp.als_sweep(Zd, dims, Ad, cp.norm2(Zd, dims)))
    _, oo = oracle.als_sweep(Z, dims, A)
    assert out[2] == cp.CP_ENOTSPD == oo[2]
    assert out[3] == oo[3] == 0
    assert math.isnan(out[0])


@pytest.mark.parametrize("dims,R,F", [((4, 4, 4), 3, False), ((7, 7, 7), 3, True), ((13, 13, 13), 5, True),
                                      ((25, 25, 25), 3, True), ((9, 8, 7, 6), 4, False), ((6, 5, 4, 3, 2), 3, True),
                                      ((60, 40), 16, True), ((12, 12, 12), 32, False), ((64, 64), 32, True),
                                      ((1024, 4), 2, False)])
def test_fused_small_multi_sweep_vs_oracle(dims, R, F):
    """cp_als_sweeps: nu sweeps in ONE launch of the fused shared-memory kernel (the coarse-level
    relaxations of the multigrid cycles, Table 1 nu_c = 50) against nu oracle sweeps (P:121,
    eq:relaxinnersolve); then a call on the general path (CP_SMALL_SWEEP=0) from the same state
    agrees with the oracle too."""
    Z, A = cpsynth.random_problem(dims, R, seed=500 + R)
    if not _well_posed(dims, R):
        pytest.skip("Gamma singular for every iterate")
    nz2 = float(np.vdot(Z, Z))
    Fh = [0.05 * cpsynth.random_matrix(I, R, 7 + k) for k, I in enumerate(dims)] if F else None
    Zd, Ad = dev_problem(Z, A)
    Fd = None if Fh is None else [dev_factor(f) for f in Fh]
    nzd = cp.norm2(Zd, dims)
    nu = 7
    out = host_tensor(cp.als_sweep(Zd, dims, Ad, nzd, F=Fd, nsweeps=nu))
    assert cp.last_launch_count() == 1
    Ao = [a.copy(order="F") for a in A]
    for _ in range(nu):
        Ao, oo = oracle.als_sweep(Z, dims, Ao, F=Fh, normZ2=nz2)
    _check_sweep([host_factor(a) for a in Ad], out, Ao, oo, nz2)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_multi_sweep_call_general_path_vs_oracle(name):
    """cp_als_sweeps on tensors above the single-CTA fused-kernel limit (P > 16384): nu = 3
    sweeps in one call on the general multi-kernel path equal 3 oracle sweeps, F included."""
    d = config(name)
    dims, Z, A = d["dims"], d["Z"], d["A0"]
    R = A[0].shape[1]
    nz2 = float(np.vdot(Z, Z))
    Fh = [0.01 * cpsynth.random_matrix(I, R, 30 + k) for k, I in enumerate(dims)]
    Zd, Ad = dev_problem(Z, A)
    out = host_tensor(cp.als_sweep(Zd, dims, Ad, cp.norm2(Zd, dims), F=[dev_factor(f) for f in Fh], nsweeps=3))
    assert cp.last_launch_count() > 3
    Ao = [a.copy(order="F") for a in A]
    for _ in range(3):
        Ao, oo = oracle.als_sweep(Z, dims, Ao, F=Fh, normZ2=nz2)
    _check_sweep([host_factor(a) for a in Ad], out, Ao, oo, nz2)


@pytest.mark.parametrize("dims,R,F", [((40, 36, 30), 20, True), ((30, 28, 26, 12), 6, True), ((33, 2), 5, False),
                                      ((64, 9, 7, 5, 3), 4, True), ((130, 9, 6), 20, False)])
def test_multi_sweep_steady_state_vs_oracle(dims, R, F, monkeypatch):
    """cp_als_sweeps on the general path: sweeps k >= 1 of one call run steady-state (no prep
    launch; the previous sweep's At copies and Gram totals) -- the tree sweep (N = 3, 4, 5: Y_R
    path), the N = 2 mode-by-mode sweep and an MMA k-split shape; nu = 4 sweeps equal 4 oracle
    sweeps, F included, and fewer launches than 4 separate calls."""
    monkeypatch.setenv("CP_SMALL_SWEEP", "0")
    Z, A = cpsynth.random_problem(dims, R, seed=900 + R)
    if not _well_posed(dims, R):
        pytest.skip("Gamma singular for every iterate")
    nz2 = float(np.vdot(Z, Z))
    Fh = [0.02 * cpsynth.random_matrix(I, R, 40 + k) for k, I in enumerate(dims)] if F else None
    Zd, Ad = dev_problem(Z, A)
    Fd = None if Fh is None else [dev_factor(f) for f in Fh]
    nzd = cp.norm2(Zd, dims)
    out = host_tensor(cp.als_sweep(Zd, dims, Ad, nzd, F=Fd, nsweeps=4))
    n4 = cp.last_launch_count()
    cp.als_sweep(Zd, dims, [a.clone() for a in Ad], nzd, F=Fd)
    n1 = cp.last_launch_count()
    # the prep launch of sweeps 2..4 is gone; N = 3 tensor-core plans also solve the last mode of
    # sweeps 1..3 inside the pass (tests/test_gpu_sweep_tail.py)
    assert n4 == 4 * n1 - 3 or (len(dims) == 3 and n4 == 4 * n1 - 6)
    Ao = [a.copy(order="F") for a in A]
    for _ in range(4):
        Ao, oo = oracle.als_sweep(Z, dims, Ao, F=Fh, normZ2=nz2)
    _check_sweep([host_factor(a) for a in Ad], out, Ao, oo, nz2)


@pytest.mark.parametrize("dims,R", [((7, 7, 7), 3), ((13, 12, 11), 4), ((50, 50, 50), 3), ((9, 8, 7, 6), 2)])
@pytest.mark.parametrize("small", ["1", "0"])
def test_multi_sweep_normalized_vs_oracle(dims, R, small, monkeypatch):
    """cp_als_sweeps with CP_SWEEPS_NORMALIZE (the setup-phase ALS relaxation: every sweep followed
    by eq:ALSnorm without sorting) against nu oracle sweeps + oracle normalizations, on
    the fused path and on the general path (sweep + cp_normalize_sort launches); f, f~ are the last
    sweep's, before its normalization."""
    monkeypatch.setenv("CP_SMALL_SWEEP", small)
    Z, A = cpsynth.random_problem(dims, R, seed=700 + R)
    nz2 = float(np.vdot(Z, Z))
    Zd, Ad = dev_problem(Z, A)
    nu = 4
    out = host_tensor(cp.als_sweep(Zd, dims, Ad, cp.norm2(Zd, dims), nsweeps=nu, normalize=True))
    Ao = [a.copy(order="F") for a in A]
    for _ in range(nu):
        Ao, oo = oracle.als_sweep(Z, dims, Ao, normZ2=nz2)
        Ao, _ = oracle.normalize_sort(dims, Ao, sort=False)
    _check_sweep([host_factor(a) for a in Ad], out, Ao, oo, nz2)


@pytest.mark.parametrize("R", [2, 8])
@pytest.mark.parametrize("small", ["1", "0"])
def test_multi_sweep_reports_enotspd_mid_run(R, small, monkeypatch):
    """Z = 0: the mode-0 update gives A^(0) = 0, so Gamma^(1) = 0 is singular in the first sweep of
    a multi-sweep call: status CP_ENOTSPD, failed mode 1, f = NaN -- as the oracle reports
    (R = 2: one-thread Cholesky; R = 8: warp Cholesky) -- on the fused path and on the general
    path, where the later sweeps of the call must neither clear the status nor touch the factors
    (they equal the oracle's after its failing sweep)."""
    monkeypatch.setenv("CP_SMALL_SWEEP", small)
    dims = (6, 5, 4) if small == "1" else (40, 30, 20)
    _, A = cpsynth.random_problem(dims, R, seed=9)
    Z = np.zeros(tuple(reversed(dims)))
    Zd, Ad = dev_problem(Z, A)
    out = host_tensor(cp.als_sweep(Zd, dims, Ad, cp.norm2(Zd, dims), nsweeps=5))
    Ao, oo = oracle.als_sweep(Z, dims, A)
    assert out[2] == cp.CP_ENOTSPD == oo[2]
    assert out[3] == oo[3] == 1
    assert math.isnan(out[0])
    for a, b in zip(Ad, Ao):
        np.testing.assert_array_equal(host_factor(a), b)


def test_sweep_rank1_exact():
    dims = (16, 12, 10)
    Z, _, A0 = cpsynth.lowrank_problem(dims, 1, seed=1)
    Zd, Ad = dev_problem(Z, A0)
    out = host_tensor(cp.als_sweep(Zd, dims, Ad, cp.norm2(Zd, dims)))
    X = cpsynth.kruskal([host_factor(a) for a in Ad])
    assert relerr(X, Z) <= 1e-13
    assert abs(out[0]) <= 1e-14 * 0.5 * float(np.vdot(Z, Z))


def test_sweep_deterministic():
    d = config("c2")
    dims = d["dims"]
    res = []
    for _ in range(2):
        Zd, Ad = dev_problem(d["Z"], d["A0"])
        nzd = cp.norm2(Zd, dims)
        for _ in range(3):
            out = cp.als_sweep(Zd, dims, Ad, nzd)
        res.append(([host_factor(a) for a in Ad], host_tensor(out)))
    for a, b in zip(res[0][0], res[1][0]):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(res[0][1], res[1][1])


# ------------------------------------------------------------------------------- mode products
@pytest.mark.parametrize("dims,J", [((5, 4, 3), 2), ((7, 6, 5), 9), ((20, 20, 20), 10), ((3, 3, 3, 3), 4),
                                    ((130, 70), 65), ((9,), 4), ((65, 3, 67), 33)])
def test_mode_product_ragged(dims, J):
    Z, _ = cpsynth.random_problem(dims, 1, seed=sum(dims))
    Zd = dev_tensor(Z)
    for n in range(len(dims)):
        U = cpsynth.random_matrix(J, dims[n], seed=n + 3)
        X, nd = cp.mode_product(Zd, dims, n, dev_factor(U))
        Xo, ndo = oracle.mode_product(Z, dims, n, U)
        assert nd == ndo
        assert relerr(host_tensor(X), Xo) <= 1e-12, (dims, J, n)


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3"])
def test_restriction_configs(name):
    """Restriction Z x_n Phat^T with a dense orthonormal Phat (c3: 256 x 128), every mode."""
    d = config(name)
    dims, Z = d["dims"], d["Z"]
    Zd = dev_tensor(Z)
    for n in range(len(dims)):
        U = np.asfortranarray(d["Phat"][n].T)
        X, nd = cp.mode_product(Zd, dims, n, dev_factor(U))
        Xo, _ = oracle.mode_product(Z, dims, n, U)
        assert relerr(host_tensor(X), Xo) <= 1e-12, (name, n)


@pytest.mark.parametrize("name", ["c4a", "c4b"])
def test_restriction_full_size_sampled_fibers(name):
    """Restriction at full size (c4a 512^3 -> 256 along the mode; c4b 96^4 -> 48): the whole
    output on the GPU, 32 sampled output fibers per mode against Phat^T applied on the host."""
    d = config(name)
    dims, Z = d["dims"], d["Z"]
    N = len(dims)
    Zt = Z.reshape(tuple(reversed(dims)))
    Zd = dev_tensor(Z)
    rng = np.random.default_rng(17)
    for n in range(N):
        U = np.asfortranarray(d["Phat"][n].T)
        X, nd = cp.mode_product(Zd, dims, n, dev_factor(U))
        Xt = host_tensor(X).reshape(tuple(reversed(nd)))
        ax = N - 1 - n
        for _ in range(32):
            idx = [int(rng.integers(0, m)) for m in reversed(dims)]
            sl = tuple(slice(None) if a == ax else idx[a] for a in range(N))
            assert relerr(Xt[sl], U @ Zt[sl]) <= 1e-12, (name, n)
        del X


def test_interpolation_factor_matrix():
    """Interpolation A = Phat A_c (eq:CGC) = cp_mode_product on the 2-way factor matrix."""
    I, Ic, R = 50, 25, 3
    Ph = cpsynth.random_matrix(I, Ic, 1)
    Ac = cpsynth.random_matrix(Ic, R, 2)
    X, nd = cp.mode_product(dev_tensor(np.ascontiguousarray(Ac.T)), (Ic, R), 0, dev_factor(Ph))
    assert nd == [I, R]
    assert relerr(host_tensor(X).T, Ph @ Ac) <= 1e-13


# ------------------------------------------------------------------------------- fit
@pytest.mark.parametrize("dims,R", [((5, 7, 3), 3), ((20, 20, 20), 3), ((2, 3, 2, 3), 2), ((700, 5, 4), 16),
                                    ((33, 2), 5)])
def test_fit_ragged(dims, R):
    Z, A = cpsynth.random_problem(dims, R, seed=R + 50)
    F = [0.1 * cpsynth.random_matrix(I, R, k) for k, I in enumerate(dims)]
    for Fuse in (None, F):
        Zd, Ad = dev_problem(Z, A)
        Fd = None if Fuse is None else [dev_factor(f) for f in Fuse]
        out, G = cp.fit(Zd, dims, Ad, cp.norm2(Zd, dims), F=Fd, want_G=True)
        out = host_tensor(out)
        oo, Go = oracle.gradient(Z, dims, A, F=Fuse)
        assert abs(out[0] - oo[0]) <= 1e-12 * abs(oo[0]) + 1e-14 * float(np.vdot(Z, Z))
        assert abs(out[1] - oo[1]) <= 1e-10 * abs(oo[1]) + 1e-13
        for n in range(len(dims)):
            assert relerr(host_factor(G[n]), Go[n]) <= 1e-11
            assert abs(out[2 + n] - oo[2 + n]) <= 1e-10 * oo[2 + n] + 1e-24


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3", "c4a", "c4b"])
def test_fit_configs(name):
    """cp_fit (a8): the direct f of the residual pass against oracle_f_direct (the plain definition
    1/2 ||Z - [[A]]||^2, eq:CPfunctional) and g against oracle_gradient, on every config -- the
    full sizes included (bench launch configuration)."""
    d = config(name)
    dims, Z, A = d["dims"], d["Z"], d["A0"]
    Zd, Ad = dev_problem(Z, A)
    out = host_tensor(cp.fit(Zd, dims, Ad, cp.norm2(Zd, dims))[0])
    del Zd
    oo, _ = oracle.gradient(Z, dims, A, want_G=False)
    assert abs(out[0] - oo[0]) <= 1e-12 * abs(oo[0])
    assert abs(out[1] - oo[1]) <= 1e-10 * abs(oo[1]) + 1e-13
    for n in range(len(dims)):
        assert abs(out[2 + n] - oo[2 + n]) <= 1e-10 * oo[2 + n]


@pytest.mark.parametrize("dims,R", [((5, 7, 3), 3), ((20, 20, 20), 3), ((2, 3, 2, 3), 2), ((700, 5, 4), 16),
                                    ((33, 29, 31), 16), ((9, 8, 7, 6), 5), ((11, 13), 4), ((6, 5, 4, 3, 2), 3)])
def test_gradient_ragged(dims, R, monkeypatch):
    """cp_gradient: g, ||G^(n)||^2, G against the oracle's gradient (eq:gradEqn,
    eq:gradConv) and f against the oracle's expansion (reading R6), on both paths (small tensors:
    the fused shared-memory kernel in gradient mode); on the general path (CP_SMALL_SWEEP=0) g and
    G are bitwise cp_fit's (same kernels, same order: only the residual pass is dropped)."""
    Z, A = cpsynth.random_problem(dims, R, seed=R + 60)
    F = [0.1 * cpsynth.random_matrix(I, R, k) for k, I in enumerate(dims)]
    half = 0.5 * float(np.vdot(Z, Z))
    for path in ("1", "0"):
        monkeypatch.setenv("CP_SMALL_SWEEP", path)
        for Fuse in (None, F):
            Zd, Ad = dev_problem(Z, A)
            Fd = None if Fuse is None else [dev_factor(f) for f in Fuse]
            nz = cp.norm2(Zd, dims)
            out, G = cp.gradient(Zd, dims, Ad, nz, F=Fd, want_G=True)
            outf, Gf = cp.fit(Zd, dims, Ad, nz, F=Fd, want_G=True)
            out, outf = host_tensor(out), host_tensor(outf)
            oo, Go = oracle.gradient(Z, dims, A, F=Fuse)
            fe = oracle.f_expand(Z, dims, A)
            assert abs(out[0] - fe) <= 1e-10 * abs(fe) + 1e-14 * half
            assert abs(out[1] - oo[1]) <= 1e-10 * abs(oo[1]) + 1e-13
            if path == "0":
                assert np.array_equal(out[1:], outf[1:])
            for n in range(len(dims)):
                g = host_factor(G[n])
                assert relerr(g, Go[n]) <= 1e-11
                if path == "0":
                    assert np.array_equal(g, host_factor(Gf[n]))
                assert abs(out[2 + n] - oo[2 + n]) <= 1e-10 * oo[2 + n] + 1e-24


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3"])
def test_gradient_configs(name):
    d = config(name)
    dims, Z, A = d["dims"], d["Z"], d["A0"]
    Zd, Ad = dev_problem(Z, A)
    out = host_tensor(cp.gradient(Zd, dims, Ad, cp.norm2(Zd, dims))[0])
    oo, _ = oracle.gradient(Z, dims, A, want_G=False)
    fe = oracle.f_expand(Z, dims, A)
    assert abs(out[0] - fe) <= 1e-10 * abs(fe) + 1e-14 * 0.5 * float(np.vdot(Z, Z))
    assert abs(out[1] - oo[1]) <= 1e-10 * abs(oo[1]) + 1e-13
    for n in range(len(dims)):
        assert abs(out[2 + n] - oo[2 + n]) <= 1e-10 * oo[2 + n]


@pytest.mark.parametrize("name", ["c4a", "c4b"])
def test_gradient_full_size_matches_fit(name):
    """At the full sizes: g, ||G^(n)||^2 bitwise cp_fit's (whose parity against the oracle is
    test_fit_configs); f (expansion) within cancellation of cp_fit's direct f."""
    d = config(name)
    dims, Z, A = d["dims"], d["Z"], d["A0"]
    Zd, Ad = dev_problem(Z, A)
    nz = cp.norm2(Zd, dims)
    out = host_tensor(cp.gradient(Zd, dims, Ad, nz)[0])
    outf = host_tensor(cp.fit(Zd, dims, Ad, nz)[0])
    assert np.array_equal(out[1:], outf[1:])
    assert abs(out[0] - outf[0]) <= 1e-10 * abs(outf[0]) + 1e-13 * 0.5 * float(np.vdot(Z, Z))


def test_chained_calls_without_sync_match_synced():
    """Every kernel reads its inputs only after its programmatic-dependent-launch wait: a chain of
    library calls on one stream with no host synchronization (sweep -> restriction -> mode
    product -> fit -> MTTKRP, each consuming the previous outputs) equals the same chain with a
    synchronization after every call, bitwise."""
    dims, R = (40, 36, 30), 6
    Z, A0 = cpsynth.random_problem(dims, R, seed=77)
    wl, wr = cpsynth.transfer_weights(dims[1], seed=5)
    U = np.asfortranarray(cpsynth.random_matrix(12, dims[2], seed=6))

    def chain(sync):
        # stale NaN bit patterns in the memory the caching allocator hands out next: a kernel
        # that multiplies unwritten padding by zero instead of selecting shows up as NaN
        junk = torch.full((64 << 20,), 0xFF, dtype=torch.uint8, device="cuda")
        del junk
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

    for a, b in zip(chain(False), chain(True)):
        assert np.all(np.isfinite(a))
        assert np.array_equal(a, b)


@pytest.mark.parametrize("dims,R", [((64, 48, 40), 16), ((130, 9, 6), 20), ((30, 28, 26, 12), 6), ((96, 50, 33), 3)])
def test_lean_stream_kernels_bitwise(dims, R, monkeypatch):
    """The feature-free instantiations of the tensor-core streaming kernel (what large tensors
    run: no pre-wait prefetch, no in-pass tail) against the full-feature ones (CP_STREAM_LEAN=0)
    on the same plans: the same arithmetic, so sweep, fit and gradient agree bitwise; and the
    lean sweep against the oracle."""
    monkeypatch.setenv("CP_SMALL_SWEEP", "0")
    monkeypatch.setenv("CP_STREAM_PREFETCH", "0")
    monkeypatch.setenv("CP_SWEEP_TAIL", "0")
    Z, A = cpsynth.random_problem(dims, R, seed=77 + R)
    nz2 = float(np.vdot(Z, Z))
    Zd, _ = dev_problem(Z, A)
    nzd = cp.norm2(Zd, dims)
    res = {}
    for lean in ("1", "0"):
        monkeypatch.setenv("CP_STREAM_LEAN", lean)
        Ad = [dev_factor(a) for a in A]
        out = host_tensor(cp.als_sweep(Zd, dims, Ad, nzd, nsweeps=2))
        fit = host_tensor(cp.fit(Zd, dims, Ad, nzd)[0])
        g, G = cp.gradient(Zd, dims, Ad, nzd, want_G=True)
        res[lean] = ([host_factor(a) for a in Ad], out, fit, host_tensor(g), [host_factor(x) for x in G])
    for a, b in zip(res["1"][0] + res["1"][4], res["0"][0] + res["0"][4]):
        assert np.array_equal(a, b)
    for k in (1, 2, 3):
        assert np.array_equal(res["1"][k], res["0"][k])
    Ao = [a.copy(order="F") for a in A]
    for _ in range(2):
        Ao, oo = oracle.als_sweep(Z, dims, Ao, normZ2=nz2)
    _check_sweep(res["1"][0], res["1"][1], Ao, oo, nz2)
