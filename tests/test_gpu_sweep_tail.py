"""The sweep's last solve inside the last streaming pass (TailSolve, stream_mma.cuh sweep_tail;
N = 3 dimension-tree sweeps on the tensor-core plans): the last contributor of each segment i_2
solves row i_2 of A^(2) (eq:relaxinnersolve P:356-358, reading R1) and the last CTA of the grid
forms Upsilon^(2) and f, f~ (readings R5, R6) -- no solve launch after the pass.

CP_SWEEP_TAIL = 2: every sweep; 1 (default): only sweeps followed by another steady sweep of the
same cp_als_sweeps call, and those leave Upsilon^(2) to the next sweep's Gamma^(0) job and skip f
(TailSolve::fin = 0); 0: never.

The row solves keep the term order of solve_kernel_t, so after ONE sweep the factors must be
BITWISE equal to CP_SWEEP_TAIL=0 (pass + solve launch); f and f~ sum the same terms in another
fixed order (rounding-level difference).  Also: one launch fewer, completion words that the last
user resets (garbage-filled workspace, CUDA-graph replays), and bitwise run-to-run determinism
although the CTA that runs a solve varies."""
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
    ((20, 20, 20), 3),
    ((130, 9, 6), 20),       # NT = 3
    ((258, 7, 5), 25),       # two row blocks: 2 contributors per (CTA column group, segment)
    ((40, 36, 30), 20),      # k-split groups
    ((96, 10, 12), 24),
    ((1030, 4, 3), 7),       # I1 > 512: row blocks
    ((8, 8, 8), 32),         # R = CP_MAX_R: 4 Gram entries per thread in the finalize
    ((50, 50, 50), 3),
    ((64, 40, 700), 6),      # I_2 > the consumers' thread count: strided row-dot sums
    ((256, 256, 256), 8),    # c3 geometry: 296 CTAs, segments shared by 2 CTAs
    ((512, 64, 96), 16),     # c4a-like rows (RB = 2) at a small size
]


def _bits(t):
    return t.detach().contiguous().view(torch.int64).cpu().numpy()


def _run(Zd, dims, A, nz, F, tail, monkeypatch, nsweeps=1, ws=None):
    monkeypatch.setenv("CP_SMALL_SWEEP", "0")
    monkeypatch.setenv("CP_SWEEP_TAIL", tail)
    Ad = [dev_factor(a) for a in A]
    Fd = None if F is None else [dev_factor(f) if f is not None else None for f in F]
    out = cp.als_sweep(Zd, dims, Ad, nz, F=Fd, ws=ws, nsweeps=nsweeps)
    return Ad, host_tensor(out), cp.last_launch_count()


@pytest.mark.parametrize("with_F", [False, True])
@pytest.mark.parametrize("dims,R", SHAPES)
def test_tail_factors_bitwise_equal_solve_launch(dims, R, with_F, monkeypatch):
    Z, A = cpsynth.random_problem(dims, R, seed=40 + R)
    F = [0.05 * cpsynth.random_matrix(dims[k], R, 7 + k) if k != 0 else None for k in range(3)] if with_F else None
    Zd = dev_tensor(Z)
    nz = cp.norm2(Zd, dims)
    A0, o0, l0 = _run(Zd, dims, A, nz, F, "0", monkeypatch)
    A1, o1, l1 = _run(Zd, dims, A, nz, F, "2", monkeypatch)
    # (R = 32 on a tiny tensor: the Z ring is too small for the tail's Gram tiles -> solve launch)
    assert l1 == l0 - 1 or (R == 32 and l1 == l0), (l0, l1)
    for k in range(3):
        assert np.array_equal(_bits(A0[k]), _bits(A1[k])), (dims, R, k)
    assert o0[2] == o1[2] == 0 and o0[3] == o1[3] == -1
    nz2 = float(np.vdot(Z, Z))
    for j in (0, 1):
        assert abs(o0[j] - o1[j]) <= 1e-13 * abs(o0[j]) + 1e-15 * nz2, (j, o0, o1)
    # and against the oracle
    Ao, oo = oracle.als_sweep(Z, dims, A, F=F, normZ2=nz2)
    for k in range(3):
        assert relerr(host_factor(A1[k]), Ao[k]) <= 1e-10
    assert abs(o1[0] - oo[0]) <= 1e-10 * abs(oo[0]) + 1e-14 * 0.5 * nz2
    assert abs(o1[1] - oo[1]) <= 1e-10 * abs(oo[1]) + 1e-14 * 0.5 * nz2


@pytest.mark.parametrize("sel", ["1", "2"])
@pytest.mark.parametrize("with_F", [False, True])
@pytest.mark.parametrize("dims,R", [((40, 36, 30), 20), ((256, 256, 256), 8), ((130, 9, 6), 20), ((50, 50, 50), 3),
                                    ((512, 64, 96), 16)])
def test_tail_multi_sweep_steady_state(dims, R, with_F, sel, monkeypatch):
    """cp_als_sweeps(nsweeps = 4): sweeps 1..3 defer Upsilon^(2) to the next sweep's Gamma^(0) job
    (formed from the At^(2) rows the tail wrote) and skip f; the last sweep runs the solve launch
    (sel = 1) or the finalizing tail (sel = 2)."""
    Z, A = cpsynth.random_problem(dims, R, seed=3)
    F = [0.05 * cpsynth.random_matrix(dims[k], R, 7 + k) for k in range(3)] if with_F else None
    Zd = dev_tensor(Z)
    nz = cp.norm2(Zd, dims)
    A0, o0, l0 = _run(Zd, dims, A, nz, F, "0", monkeypatch, nsweeps=4)
    A1, o1, l1 = _run(Zd, dims, A, nz, F, sel, monkeypatch, nsweeps=4)
    assert l1 == l0 - (3 if sel == "1" else 4)
    # the Gram total of A^(2) enters Gamma^(0) of the next sweep in a different summation order:
    # rounding-level differences from sweep 2 on
    for k in range(3):
        assert relerr(host_factor(A1[k]), host_factor(A0[k])) <= 1e-12
    Ao = A
    nz2 = float(np.vdot(Z, Z))
    for _ in range(4):
        Ao, oo = oracle.als_sweep(Z, dims, Ao, F=F, normZ2=nz2)
    for k in range(3):
        assert relerr(host_factor(A1[k]), Ao[k]) <= 1e-10
    assert o1[2] == 0
    assert abs(o1[0] - oo[0]) <= 1e-10 * abs(oo[0]) + 1e-14 * 0.5 * nz2
    assert abs(o1[1] - oo[1]) <= 1e-10 * abs(oo[1]) + 1e-14 * 0.5 * nz2


@pytest.mark.parametrize("fill", [0x00, 0xFF, 0x7F, 0x5A])
def test_tail_garbage_workspace_and_determinism(fill, monkeypatch):
    dims, R = (256, 256, 256), 8
    Z, A = cpsynth.random_problem(dims, R, seed=2)
    Zd = dev_tensor(Z)
    nz = cp.norm2(Zd, dims)
    ws = cp.Workspace(dims, R)
    Aref, oref, _ = _run(Zd, dims, A, nz, None, "2", monkeypatch, ws=ws, nsweeps=3)
    for rep in range(3):
        ws.buf.fill_(fill)
        A1, o1, _ = _run(Zd, dims, A, nz, None, "2", monkeypatch, ws=ws, nsweeps=3)
        for k in range(3):
            assert np.array_equal(_bits(A1[k]), _bits(Aref[k])), (fill, rep, k)
        assert np.array_equal(o1.view(np.int64), oref.view(np.int64)), (fill, rep)


def test_tail_graph_replays(monkeypatch):
    """A captured sweep replays one launch tag: every replay must complete (segment tickets, the
    grid ticket and the Gamma-job flag are reset by their last users) and track new data."""
    monkeypatch.setenv("CP_SMALL_SWEEP", "0")
    monkeypatch.setenv("CP_SWEEP_TAIL", "2")
    dims, R = (128, 96, 80), 12
    Z, A = cpsynth.random_problem(dims, R, seed=9)
    Zd = dev_tensor(Z)
    Ad = [dev_factor(a) for a in A]
    Astart = [a.clone() for a in Ad]
    ws = cp.Workspace(dims, R)
    nz = cp.norm2(Zd, dims)
    out = torch.zeros(4, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        cp.als_sweep(Zd, dims, Ad, nz, out=out, ws=ws, stream=s, nsweeps=3)  # warm-up outside capture
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cp.als_sweep(Zd, dims, Ad, nz, out=out, ws=ws, stream=torch.cuda.current_stream(), nsweeps=3)
    rng = np.random.default_rng(4)
    for rep in range(4):
        Zn = rng.standard_normal(Z.shape)
        Zd.copy_(torch.from_numpy(Zn))
        for a, b in zip(Ad, Astart):
            a.copy_(b)
        nz.copy_(cp.norm2(Zd, dims))
        g.replay()
        torch.cuda.synchronize()
        Ar = [b.clone() for b in Astart]
        oref = cp.als_sweep(Zd, dims, Ar, nz, ws=cp.Workspace(dims, R), nsweeps=3)
        for k in range(3):
            assert np.array_equal(_bits(Ad[k]), _bits(Ar[k])), (rep, k)
        assert np.array_equal(_bits(out), _bits(oref)), rep


def test_tail_skips_after_an_earlier_mode_failed(monkeypatch):
    """Gamma^(0) singular (zero column in A^(1)): the tail must not solve, and its finalize reports
    CP_ENOTSPD with the failing mode, like the solve-launch path and the oracle."""
    dims, R = (40, 36, 30), 4
    Z, A = cpsynth.random_problem(dims, R, seed=9)
    A[1][:, 2] = 0.0
    Zd = dev_tensor(Z)
    nz = cp.norm2(Zd, dims)
    A1, o1, _ = _run(Zd, dims, A, nz, None, "2", monkeypatch, nsweeps=2)
    _, oo = oracle.als_sweep(Z, dims, A)
    assert o1[2] == cp.CP_ENOTSPD == oo[2] and o1[3] == oo[3] == 0
    assert math.isnan(o1[0]) and math.isnan(o1[1])
    assert np.array_equal(_bits(A1[2]), _bits(dev_factor(A[2])))  # A^(2) untouched
