"""Pins for the structured-restriction oracle (oracle/mg.py restrict_structured):
the transfer operator built from given F-row weights has the paper's properties (orthonormal
columns; same range as P), closed forms for I = 1, 2, and restriction followed by
interpolation reproduces tensors whose mode-n fibers lie in range(P).  No GPU needed."""
import numpy as np
import pytest

import cpsynth
import oracle
from oracle import mg


def weights(I, seed):
    return cpsynth.transfer_weights(I, seed)


@pytest.mark.parametrize("I", [1, 2, 3, 4, 9, 16, 33])
def test_interpolation_pattern_and_phat(I):
    wl, wr = weights(I, I)
    P = mg.interpolation_from_weights(I, wl, wr)
    Ic = (I + 1) // 2
    assert P.shape == (I, Ic)
    for i in range(I):
        nz = np.nonzero(P[i])[0].tolist()
        if i % 2 == 0:
            assert nz == [i // 2] and P[i, i // 2] == 1.0          # C point injected
        else:
            assert nz == ([(i - 1) // 2, (i + 1) // 2] if i + 1 < I else [(i - 1) // 2])
    Ph = mg.transfer(P)
    np.testing.assert_allclose(Ph.T @ Ph, np.eye(Ic), atol=1e-13)
    np.testing.assert_allclose(Ph @ (Ph.T @ P), P, atol=1e-13)      # range(Phat) = range(P)


def test_closed_forms_small():
    Z, _ = cpsynth.random_problem((2, 3, 4), 1, seed=7)
    wl, wr = np.array([0.0, 0.3]), np.array([0.0, 0.9])
    X, nd = mg.restrict_structured(Z, (2, 3, 4), 0, wl, wr)   # I = 2: x = (z0 + wl1 z1)/sqrt(1+wl1^2)
    assert nd == [1, 3, 4]
    Zt = Z.reshape(4, 3, 2)
    np.testing.assert_allclose(X.reshape(4, 3), (Zt[..., 0] + 0.3 * Zt[..., 1]) / np.sqrt(1.09), rtol=1e-14)
    X1, nd1 = mg.restrict_structured(Z.reshape(-1), (24,), 0, *weights(24, 1))
    assert nd1 == [12]
    Zs, _ = cpsynth.random_problem((1, 5), 1, seed=8)
    Xs, nds = mg.restrict_structured(Zs, (1, 5), 0, np.zeros(1), np.zeros(1))  # I = 1: identity
    assert nds == [1, 5]
    np.testing.assert_allclose(Xs.reshape(-1), Zs.reshape(-1), rtol=0, atol=0)


@pytest.mark.parametrize("dims,mode", [((9, 6, 5), 0), ((7, 10, 3), 1), ((4, 5, 12), 2), ((6, 8, 3, 5), 1)])
def test_restrict_then_interpolate_reproduces_range_of_P(dims, mode):
    """Z = Xc x_mode P has fibers in range(P); Phat Phat^T is the orthogonal projector onto
    range(P), so (Z x_mode Phat^T) x_mode Phat = Z."""
    I = dims[mode]
    wl, wr = weights(I, 11 + mode)
    P = mg.interpolation_from_weights(I, wl, wr)
    cd = list(dims)
    cd[mode] = P.shape[1]
    Xc, _ = cpsynth.random_problem(tuple(cd), 1, seed=3)
    Z, zd = oracle.mode_product(Xc, cd, mode, np.asfortranarray(P))
    assert list(zd) == list(dims)
    X, nd = mg.restrict_structured(Z, dims, mode, wl, wr)
    Ph = mg.transfer(P)
    Zr, _ = oracle.mode_product(X, nd, mode, Ph)
    np.testing.assert_allclose(Zr, Z, rtol=1e-12, atol=1e-12 * np.abs(Z).max())
