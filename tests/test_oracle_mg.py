"""Pins for the multigrid oracle (oracle/mg.py): structural facts of the paper's transfer
operators, the level counts of Table 4, the FAS fixed point, and convergence on the paper's
dense test problem.  No GPU needed."""
import json
import os

import numpy as np
import pytest

import cpsynth
import oracle
from oracle import mg


def test_level_counts_match_table4(golden_dir):
    rows = json.load(open(os.path.join(golden_dir, "table4_levels.json")))["rows"]
    for r in rows:
        assert len(mg.levels((r["s"],) * 3, r["R"])) == r["levs"], r


def test_coarse_sizes_odd_points():
    """C = odd points (1-based) so I_c = ceil(I/2): 5 -> 3, 4 -> 2, 2 -> 1."""
    for I, Ic in [(5, 3), (4, 2), (2, 1), (50, 25), (7, 4)]:
        U = [cpsynth.random_matrix(I, 3, 1), cpsynth.random_matrix(I, 3, 2)]
        P = mg.interpolation_matrix(U, [1.0, 1.0])
        assert P.shape == (I, Ic)
        for c in range(Ic):
            assert P[2 * c, c] == 1.0 and np.count_nonzero(P[2 * c]) == 1


def test_phat_orthonormal_columns():
    """Phat = P L^{-T} with P^T P = L L^T has orthonormal columns."""
    for I in (9, 16, 33):
        U = [cpsynth.random_matrix(I, 3, 3), cpsynth.random_matrix(I, 3, 4)]
        Ph = mg.transfer(mg.interpolation_matrix(U, [2.0, 0.5]))
        np.testing.assert_allclose(Ph.T @ Ph, np.eye(Ph.shape[1]), atol=1e-12)


def test_linear_vectors_interpolated_exactly():
    """If every fitted vector is linear in the index, the LS weights are (1/2, 1/2) in the
    interior and P reproduces the vectors from their coarse injection (eq:LSQinterp)."""
    I = 11  # odd: no one-sided end
    i = np.arange(I, dtype=float)
    U = [np.stack([1 + 2 * i, 3 - i, 0.5 * i], axis=1), np.stack([2 + i, -1 + 0.25 * i, 4 - 3 * i], axis=1)]
    P = mg.interpolation_matrix(U, [1.0, 3.0])
    for f in range(1, I, 2):
        np.testing.assert_allclose(P[f, [(f - 1) // 2, (f + 1) // 2]], [0.5, 0.5], atol=1e-12)
    for u in U:
        np.testing.assert_allclose(P @ u[::2], u, atol=1e-12)


def test_fas_fixed_point_exact_solution():
    """An exact solution (Z = [[A*]]) is a fixed point of a CP-FAS V-cycle: relaxation keeps it
    and F_c = H_c(A~_c) makes A~_c a fixed point of the coarse problem."""
    dims, R = (12, 12, 12), 2
    Z, At, _ = cpsynth.lowrank_problem(dims, R, seed=5, C=0.3)
    At, _ = oracle.normalize_sort(dims, At)
    T0 = [cpsynth.uniform_init(dims, R, seed=20 + t) for t in range(2)]
    o = mg.MGOracle(Z, dims, R, dict(mg.DEFAULTS, nuc_setup=10))
    o.lv[0].A = [a.copy(order="F") for a in At]
    o.lv[0].T = T0
    o.setup_cycle(0, True, False)       # build the operators, boot factors untouched
    o.lv[0].A = [a.copy(order="F") for a in At]
    o.fas_cycle(0, None)
    for a, b in zip(o.lv[0].A, At):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)


@pytest.mark.parametrize("fmg", [0, 1])
def test_dense_problem_converges(fmg):
    """The paper's dense tensor, s = 20, R = 2, U(0,1) initial guesses:
    Multilevel (and Multilevel + FMG) reach g < 1e-10 (eq:stopcrit) in a handful of cycles;
    the paper reports 7 for s = 50 (Table 4 test 1)."""
    s, R = 20, 2
    dims = (s, s, s)
    Z = cpsynth.dense_inverse_norm(s)
    A0 = cpsynth.uniform_init(dims, R, seed=0)
    T0 = [cpsynth.uniform_init(dims, R, seed=10 + t) for t in range(2)]
    Af = cpsynth.uniform_init(mg.levels(dims, R)[-1], R, seed=99)
    A, rep, tr = mg.mg_solve(Z, dims, A0, T0, A_fmg=Af, use_fmg=fmg, max_cycles=40)
    assert rep["status"] == 0 and rep["g"] < 1e-10 and rep["cycles"] <= 15
    # and the minimizer is a stationary point of the plain functional
    g = oracle.gradient(Z, dims, A, want_G=False)[0][1]
    assert g < 1e-10
