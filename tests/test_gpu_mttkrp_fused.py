"""cp_mttkrp in one launch (StreamPlan::Mout, stream_mma.cuh): the pass finishes M itself --
tagged per-segment tickets (modes >= 1) or a grid barrier and a sliced sum (mode 0) -- in the
fixed summation order of the separate reduce kernels.  So the fused result must be BITWISE equal
to CP_MTTKRP_FUSED=0 (stream pass + reduce launch), and both are compared with the oracle by
test_gpu_parity.py.  Also: the tagged completion words live in uninitialized caller workspace
(garbage-filled here), are reused by successive calls of different modes, and survive CUDA-graph
replays that repeat one launch tag."""
import numpy as np
import pytest

import cpsynth
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1111_6091_b200 as cp  # noqa: E402
from gpu_util import dev_factor, dev_tensor, host_factor, relerr  # noqa: E402

SHAPES = [
    ((20, 20, 20), 3),
    ((130, 9, 6), 20),       # NT = 3
    ((258, 7, 5), 25),       # two row blocks (mode 0: RB = 2 partial slices)
    ((40, 36, 30), 20),      # k-split groups
    ((1030, 3, 2), 7),       # I1 > 512: row blocks
    ((64, 9, 7, 5, 3), 4),   # N = 5: segments of many stages and of few
    ((96, 5, 6, 7), 10),
    ((256, 256, 256), 8),    # c3 geometry: 296 CTAs, segments shared by 2 CTAs
    ((512, 64, 96), 16),     # c4a-like rows (RB = 2) at a small size
]


def _bits(t):
    return t.detach().contiguous().view(torch.int64).cpu().numpy()


def _both(Zd, dims, Ad, n, ws, monkeypatch):
    monkeypatch.setenv("CP_MTTKRP_FUSED", "0")
    M0 = cp.mttkrp(Zd, dims, Ad, n, ws=ws)
    monkeypatch.setenv("CP_MTTKRP_FUSED", "2")
    M1 = cp.mttkrp(Zd, dims, Ad, n, ws=ws)
    return M0, M1


@pytest.mark.parametrize("dims,R", SHAPES)
def test_fused_bitwise_equals_two_launch_path(dims, R, monkeypatch):
    Z, A = cpsynth.random_problem(dims, R, seed=5 + R)
    Zd, Ad = dev_tensor(Z), [dev_factor(a) for a in A]
    ws = cp.Workspace(dims, R)
    for n in range(len(dims)):
        M0, M1 = _both(Zd, dims, Ad, n, ws, monkeypatch)
        assert np.array_equal(_bits(M0), _bits(M1)), (dims, R, n)
    # one oracle check per shape on the fused result (the parity suite covers every mode)
    n = len(dims) - 1
    assert relerr(host_factor(M1), oracle.mttkrp(Z, dims, A, n)) <= 1e-12


@pytest.mark.parametrize("fused", ["1", "2"])
@pytest.mark.parametrize("fill", [0x00, 0xFF, 0x7F, 0x5A])
def test_fused_garbage_workspace_and_mode_interleaving(fill, fused, monkeypatch):
    monkeypatch.setenv("CP_MTTKRP_FUSED", fused)
    dims, R = (256, 256, 256), 8
    Z, A = cpsynth.random_problem(dims, R, seed=2)
    Zd, Ad = dev_tensor(Z), [dev_factor(a) for a in A]
    ws = cp.Workspace(dims, R)
    ref = [cp.mttkrp(Zd, dims, Ad, n, ws=ws).clone() for n in range(3)]
    ws.buf.fill_(fill)
    for n in (0, 1, 0, 2, 2, 1, 0):
        M = cp.mttkrp(Zd, dims, Ad, n, ws=ws)
        assert np.array_equal(_bits(M), _bits(ref[n])), (fill, n)


@pytest.mark.parametrize("fused", ["1", "2"])
def test_fused_graph_replays(fused, monkeypatch):
    """A captured cp_mttkrp replays one launch tag; every replay must still complete (the last
    arrival of each word resets it) and track new data."""
    monkeypatch.setenv("CP_MTTKRP_FUSED", fused)
    dims, R = (128, 96, 80), 12
    Z, A = cpsynth.random_problem(dims, R, seed=9)
    Zd, Ad = dev_tensor(Z), [dev_factor(a) for a in A]
    ws = cp.Workspace(dims, R)
    outs = [cp.empty_factor(dims[n], R, Zd.device) for n in range(3)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for n in range(3):  # warm-up outside capture (plans, tensor maps, attributes)
            cp.mttkrp(Zd, dims, Ad, n, M=outs[n], ws=ws, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for n in range(3):
            cp.mttkrp(Zd, dims, Ad, n, M=outs[n], ws=ws, stream=torch.cuda.current_stream())
    rng = np.random.default_rng(4)
    for rep in range(4):
        Zn = rng.standard_normal(Z.shape)
        Zd.copy_(torch.from_numpy(Zn))
        g.replay()
        torch.cuda.synchronize()
        for n in range(3):
            ref = cp.mttkrp(Zd, dims, Ad, n, ws=cp.Workspace(dims, R))
            assert np.array_equal(_bits(outs[n]), _bits(ref)), (rep, n)
