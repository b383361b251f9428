"""cp_als_sweeps_then_gradient: the pre-relaxation and H(A) of a CP-FAS level (Algorithm 2
P:373-420, eq:FASrhs P:398) as one call -- bitwise the results of cp_als_sweeps followed by
cp_gradient, on the fused small-tensor path (one launch), the tiny-kernel shapes and the general
path (two calls inside), with a FAS right-hand side in the sweeps and with the normalization flag."""
import numpy as np
import pytest

import cpsynth
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1111_6091_b200 as cp  # noqa: E402
from gpu_util import dev_factor, dev_tensor, host_factor  # noqa: E402


def _bits(t):
    return t.detach().contiguous().view(torch.int64).cpu().numpy()


@pytest.mark.parametrize("normalize", [False, True])
@pytest.mark.parametrize("dims,R,nu", [((25, 25, 25), 3, 1), ((13, 13, 13), 3, 2), ((7, 7, 7), 3, 1), ((4, 4, 4), 3, 3),
                                       ((9, 8, 7, 6), 4, 1), ((50, 50, 50), 3, 1), ((60, 40), 5, 2)])
def test_equals_the_two_calls_bitwise(dims, R, nu, normalize):
    Z, A = cpsynth.random_problem(dims, R, seed=11 + R)
    N = len(dims)
    F = None if normalize else [0.05 * cpsynth.random_matrix(dims[k], R, 3 + k) for k in range(N)]
    Zd = dev_tensor(Z)
    nz = cp.norm2(Zd, dims)
    Fd = None if F is None else [dev_factor(f) for f in F]
    A1 = [dev_factor(a) for a in A]
    o1 = cp.als_sweep(Zd, dims, A1, nz, F=Fd, nsweeps=nu, normalize=normalize)
    n_sep = cp.last_launch_count()
    g1, G1 = cp.gradient(Zd, dims, A1, nz, want_G=True)
    n_sep += cp.last_launch_count()
    A2 = [dev_factor(a) for a in A]
    o2, g2, G2 = cp.als_sweeps_then_gradient(Zd, dims, A2, nz, F=Fd, nsweeps=nu, normalize=normalize)
    n_one = cp.last_launch_count()
    for k in range(N):
        assert np.array_equal(_bits(A1[k]), _bits(A2[k]))
        assert np.array_equal(_bits(G1[k]), _bits(G2[k]))
    assert np.array_equal(_bits(o1), _bits(o2))
    assert np.array_equal(_bits(g1), _bits(g2))
    P = int(np.prod(dims))
    tiny = N <= 4 and R <= 4 and all(P // d <= 32 for d in dims)  # tiny_sweep.cu's shapes: two calls inside
    if P <= 16384 and not tiny:
        assert n_one == 1 and n_sep == 2  # the fused kernel ran both
    else:
        assert n_one == n_sep
    # and the gradient itself against the oracle at the new iterate
    Ah = [host_factor(a) for a in A2]
    fo, Go = oracle.gradient(Z, dims, Ah, want_G=True)
    # (G = A Gamma - M is a difference of two O(|M|) terms: after a sweep without F the last
    # mode's gradient is zero up to rounding, so the error is measured against |M|)
    for k in range(N):
        Mk = np.linalg.norm(oracle.mttkrp(Z, dims, Ah, k))
        assert np.linalg.norm(host_factor(G2[k]) - Go[k]) <= 1e-9 * np.linalg.norm(Go[k]) + 1e-12 * Mk
    assert abs(g2.cpu().numpy()[1] - fo[1]) <= 1e-10 * fo[1] + 1e-13


def test_failed_sweeps_give_nan_gradient():
    dims, R = (13, 13, 13), 3
    Z, A = cpsynth.random_problem(dims, R, seed=2)
    A[1][:, 1] = 0.0
    Zd = dev_tensor(Z)
    o, g, _ = cp.als_sweeps_then_gradient(Zd, dims, [dev_factor(a) for a in A], cp.norm2(Zd, dims))
    o, g = o.cpu().numpy(), g.cpu().numpy()
    assert o[2] == cp.CP_ENOTSPD and o[3] == 0
    assert np.isnan(g[0]) and np.isnan(g[1])
