"""Pins for the CPU oracle (oracle/cp_oracle.c) against things other than itself.

Each test states the passage of PAPER.md ("P:n") or the mathematical fact that fixes the
expected value: worked examples (tests/golden/, each with its citation), closed forms,
textbook special cases (Eckart-Young via LAPACK SVD, numpy Cholesky / eigh), invariants
(monotone f, fixed points, gradient vs finite differences) and brute force on tiny inputs
written independently of the oracle (explicit unfold + Kronecker, Python loops).
No GPU needed.
"""
import functools
import itertools
import json
import math
import os

import numpy as np
import pytest

import cpsynth
import oracle


def unfold(Z, dims, n):
    """Mode-n matricization Z_(n), columns with the lowest remaining mode fastest."""
    Zf = np.asarray(Z).reshape(cpsynth.tensor_shape(dims)).transpose(range(len(dims))[::-1])
    return np.moveaxis(Zf, n, 0).reshape(dims[n], -1, order="F")


def phi_explicit(A, n):
    """Phi^(n) = A^(N) (.) ... (.) A^(n+1) (.) A^(n-1) (.) ... (.) A^(1) (eq:Phi P:109-111),
    built column by column with numpy.kron (the Khatri-Rao definition)."""
    N = len(A)
    R = A[0].shape[1]
    cols = []
    for r in range(R):
        vecs = [A[k][:, r] for k in reversed(range(N)) if k != n]
        cols.append(functools.reduce(np.kron, vecs))
    return np.stack(cols, axis=1)


def mttkrp_loops(Z, dims, A, n):
    """Brute force: every element, every r, the product of the N-1 factor entries (no reuse)."""
    N = len(dims)
    R = A[0].shape[1]
    Zf = np.asarray(Z).reshape(cpsynth.tensor_shape(dims))
    M = np.zeros((dims[n], R))
    for idx in itertools.product(*[range(d) for d in dims]):
        z = Zf[tuple(reversed(idx))]
        for r in range(R):
            p = z
            for k in range(N):
                if k != n:
                    p *= A[k][idx[k], r]
            M[idx[n], r] += p
    return M


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


# ---------------------------------------------------------------- MTTKRP


def test_norm2_closed_forms_and_library():
    """||Z||^2 of eq:CPfunctional = sum of squared entries: (i) the all-ones tensor of
    P elements gives exactly P; (ii) a scaled unit tensor c*e_k gives c^2; (iii) integer entries
    0..P-1 give the closed form (P-1)P(2P-1)/6 exactly (every partial sum is an integer below
    2^53); (iv) random data agrees with numpy's dot product (a different summation order) to
    a few ulps.  Pins oracle_norm2 (previously "parity unpinned")."""
    for dims in [(1,), (3, 4, 2), (7, 5, 3, 2)]:
        P = int(np.prod(dims))
        assert oracle.norm2(np.ones(cpsynth.tensor_shape(dims))) == float(P)
        e = np.zeros(P)
        e[P // 2] = -3.5
        assert oracle.norm2(e) == 12.25
        v = np.arange(P, dtype=np.float64)
        assert oracle.norm2(v) == float((P - 1) * P * (2 * P - 1) // 6)
    Z, _ = cpsynth.random_problem((33, 17, 9), 1, seed=77)
    ref = float(np.dot(Z.reshape(-1), Z.reshape(-1)))
    assert abs(oracle.norm2(Z) - ref) <= 1e-13 * ref
    assert oracle.norm2(np.zeros(5)) == 0.0


def test_kr_order_worked_example(golden_dir):
    """KR ordering of Phi: the worked example A (.) B must come out of the
    oracle's mode-3 MTTKRP of a 2x2x4 tensor whose mode-3 unfolding is the identity."""
    g = json.load(open(os.path.join(golden_dir, "kr_example.json")))
    Aw, Bw, expect = np.array(g["A"], float), np.array(g["B"], float), np.array(g["A_kr_B"], float)
    dims = (2, 2, 4)
    Z = np.zeros(cpsynth.tensor_shape(dims))
    for i1 in range(2):
        for i2 in range(2):
            Z[i1 + 2 * i2, i2, i1] = 1.0   # Z_(3) = I_4 with column j = i1 + 2*i2
    C = np.asfortranarray(np.ones((4, 2)))
    # Phi^(3) = A^(2) (.) A^(1): A^(2) = Aw, A^(1) = Bw (A^(1)'s index fastest)
    M = oracle.mttkrp(Z, dims, [np.asfortranarray(Bw), np.asfortranarray(Aw), C], 2)
    np.testing.assert_array_equal(M, expect)


@pytest.mark.parametrize("dims,R", [((3, 4, 2), 2), ((2, 3, 2, 3), 3), ((5, 1, 3), 2), ((1, 4), 3)])
def test_mttkrp_bruteforce_and_explicit_phi(dims, R):
    """Brute-force elementwise MTTKRP and Z_(n) @ Phi^(n) with explicit Phi (BJ)."""
    Z, A = cpsynth.random_problem(dims, R, seed=sum(dims) + R)
    for n in range(len(dims)):
        Mo = oracle.mttkrp(Z, dims, A, n)
        Mb = mttkrp_loops(Z, dims, A, n)
        Mp = unfold(Z, dims, n) @ phi_explicit(A, n)
        assert rel(Mo, Mb) <= 1e-14
        assert rel(Mo, Mp) <= 1e-14


def test_mttkrp_zero_tensor():
    dims = (3, 4, 5)
    Z = np.zeros(cpsynth.tensor_shape(dims))
    _, A = cpsynth.random_problem(dims, 3, seed=7)
    for n in range(3):
        assert not np.any(oracle.mttkrp(Z, dims, A, n))


@pytest.mark.parametrize("dims,S,R", [((40, 30, 20), 4, 5), ((7, 9, 6, 5), 3, 4), ((64, 33), 5, 2)])
def test_mttkrp_kruskal_closed_form(dims, S, R):
    """If Z = [[U]] (rank S) then M^(n) = U^(n) (*_{k!=n} U^(k)^T A^(k)) by eq:propKKR."""
    U = [cpsynth.random_matrix(I, S, seed=10 + k) for k, I in enumerate(dims)]
    A = [cpsynth.random_matrix(I, R, seed=50 + k) for k, I in enumerate(dims)]
    Z = cpsynth.kruskal(U)
    for n in range(len(dims)):
        H = np.ones((S, R))
        for k in range(len(dims)):
            if k != n:
                H *= U[k].T @ A[k]
        assert rel(oracle.mttkrp(Z, dims, A, n), U[n] @ H) <= 1e-13


def test_mttkrp_row_subset_matches_full():
    dims = (6, 5, 7)
    Z, A = cpsynth.random_problem(dims, 3, seed=3)
    full = oracle.mttkrp(Z, dims, A, 2)
    part = oracle.mttkrp(Z, dims, A, 2, rows=(2, 5))
    np.testing.assert_array_equal(part[2:5], full[2:5])


# ---------------------------------------------------------------- Gram / Gamma / Cholesky


def test_gamma_spd_and_model_norm():
    """Gamma is a Hadamard product of SPSD Grams, hence SPSD, and
    1^T(*_k Upsilon^(k))1 = ||[[A]]||^2 (explicit reconstruction)."""
    dims = (6, 5, 4)
    _, A = cpsynth.random_problem(dims, 4, seed=11)
    Ups = [oracle.gram(a) for a in A]
    for a, u in zip(A, Ups):
        np.testing.assert_allclose(u, a.T @ a, rtol=1e-14, atol=1e-14)
    for n in range(3):
        G = np.ones((4, 4))
        for k in range(3):
            if k != n:
                G *= Ups[k]
        assert np.allclose(G, G.T, rtol=0, atol=1e-13)
        assert np.linalg.eigvalsh(G).min() >= -1e-10
    H = Ups[0] * Ups[1] * Ups[2]
    X = cpsynth.kruskal(A)
    assert abs(H.sum() - np.vdot(X, X)) <= 1e-13 * np.vdot(X, X)


def test_cholesky_and_solve_match_lapack_and_pinv():
    """Cholesky equals LAPACK's; the row solve equals post-multiplication by the
    Moore-Penrose pseudoinverse when Gamma is SPD."""
    rng = np.random.default_rng(5)
    for R in (1, 2, 5, 16, 32):
        B0 = rng.standard_normal((R + 7, R))
        G = B0.T @ B0
        st, L = oracle.cholesky(G)
        assert st == 0
        np.testing.assert_allclose(L, np.linalg.cholesky(G), rtol=1e-12, atol=1e-12)
        Bm = rng.standard_normal((9, R))
        X = oracle.solve_rows(L, Bm)
        w, V = np.linalg.eigh(G)
        pinv = (V / w) @ V.T
        cond = w.max() / w.min()
        assert rel(X, Bm @ pinv) <= 1e-15 * cond * 50
        assert rel(X @ G, Bm) <= 1e-15 * cond * 50


def test_cholesky_rejects_singular():
    G = np.array([[1.0, 1.0], [1.0, 1.0]])
    st, _ = oracle.cholesky(G)
    assert st == oracle.ENOTSPD
    st, _ = oracle.cholesky(np.zeros((3, 3)))
    assert st == oracle.ENOTSPD


# ---------------------------------------------------------------- f and gradient


def test_f_direct_special_cases():
    dims = (5, 4, 3)
    Z, A = cpsynth.random_problem(dims, 2, seed=21)
    X = cpsynth.kruskal(A)
    assert abs(oracle.f_direct(X, dims, A)) <= 1e-26 * np.vdot(X, X) + 1e-300
    zero = [np.zeros_like(a, order="F") for a in A]
    assert oracle.f_direct(Z, dims, zero) == pytest.approx(0.5 * np.vdot(Z, Z), rel=1e-15)
    assert oracle.f_direct(Z, dims, A) == pytest.approx(0.5 * np.sum((Z - X) ** 2), rel=1e-13)


@pytest.mark.parametrize("dims,R", [((5, 4, 3), 2), ((3, 2, 4, 3), 3), ((7, 6), 2), ((4, 3, 2, 2, 3), 4)])
def test_f_expand_special_cases_and_direct(dims, R):
    """oracle.f_expand (reading R6: 1/2||Z||^2 - <M^(N),A^(N)> + 1/2 1^T(*Upsilon)1) against the plain
    definition f_direct = 1/2 sum (z - x)^2 (eq:CPfunctional P:38-42) on random iterates; an exact
    model gives f = 0 up to cancellation; zero factors give 1/2||Z||^2 exactly; a dropped Gram,
    a wrong mode in the inner product or a missing factor 1/2 fails one of them."""
    Z, A = cpsynth.random_problem(dims, R, seed=41 + R)
    half = 0.5 * float(np.vdot(Z, Z))
    assert oracle.f_expand(Z, dims, A) == pytest.approx(oracle.f_direct(Z, dims, A), abs=1e-13 * half)
    X = cpsynth.kruskal(A)
    assert abs(oracle.f_expand(X, dims, A)) <= 1e-13 * 0.5 * float(np.vdot(X, X))
    zero = [np.zeros_like(a, order="F") for a in A]
    assert oracle.f_expand(Z, dims, zero) == half
    # a perturbed iterate moves f_direct and f_expand together (not a constant offset)
    B = [a.copy(order="F") for a in A]
    B[0][0, 0] += 0.3
    assert oracle.f_expand(Z, dims, B) == pytest.approx(oracle.f_direct(Z, dims, B), abs=1e-13 * half)
    assert abs(oracle.f_direct(Z, dims, B) - oracle.f_direct(Z, dims, A)) > 1e-6 * half


@pytest.mark.parametrize("dims,R", [((4, 3, 5), 2), ((3, 2, 4, 3), 3), ((6, 5, 4), 1)])
def test_gradient_vs_finite_differences(dims, R):
    """G^(n) (eq:gradEqn P:104-107) against central differences of f (eq:CPfunctional),
    h = 1e-6, relative 1e-5."""
    Z, A = cpsynth.random_problem(dims, R, seed=31 + R)
    out, G = oracle.gradient(Z, dims, A)
    h = 1e-6
    for n in range(len(dims)):
        fd = np.zeros_like(A[n])
        for i in range(dims[n]):
            for r in range(R):
                Ap = [a.copy(order="F") for a in A]
                Am = [a.copy(order="F") for a in A]
                Ap[n][i, r] += h
                Am[n][i, r] -= h
                fd[i, r] = (oracle.f_direct(Z, dims, Ap) - oracle.f_direct(Z, dims, Am)) / (2 * h)
        assert rel(G[n], fd) <= 1e-5
        assert out[2 + n] == pytest.approx(np.sum(G[n] ** 2), rel=1e-14)
    assert out[1] == pytest.approx(math.sqrt(sum(out[2:])) / np.linalg.norm(Z), rel=1e-14)


def test_gradient_with_rhs_is_fas_residual():
    """With F, G^(n) = H^(n)(A) - F^(n) (eq:FASop, eq:FASfineprob P:326-332)."""
    dims = (4, 5, 3)
    Z, A = cpsynth.random_problem(dims, 2, seed=41)
    F = [cpsynth.random_matrix(I, 2, seed=60 + k) for k, I in enumerate(dims)]
    _, G0 = oracle.gradient(Z, dims, A)
    _, G1 = oracle.gradient(Z, dims, A, F=F)
    for n in range(3):
        np.testing.assert_allclose(G1[n], G0[n] - F[n], rtol=1e-14, atol=1e-14)


# ---------------------------------------------------------------- the sweep


def test_sweep_rank1_one_step_exact():
    """Noiseless rank-1 Z: one sweep from a generic init reproduces Z exactly (each mode
    update recovers the exact direction; closed form)."""
    dims = (7, 6, 5)
    Z, At, A0 = cpsynth.lowrank_problem(dims, 1, seed=1)
    A1, out = oracle.als_sweep(Z, dims, A0)
    X = cpsynth.kruskal(A1)
    assert rel(X, Z) <= 1e-14
    # the expanded f cancels: its floor is ~eps * 1/2||Z||^2 (SURVEY 8(c) f tolerance)
    assert abs(out[0]) <= 1e-14 * 0.5 * np.vdot(Z, Z)
    assert oracle.f_direct(Z, dims, A1) <= 1e-28 * np.vdot(Z, Z)


def test_sweep_matrix_case_eckart_young():
    """N = 2: ALS converges to the best rank-R approximation, f* = 1/2 sum_{i>R} sigma_i^2
    (Eckart-Young; LAPACK SVD)."""
    rng = np.random.default_rng(9)
    I1, I2, R = 30, 20, 3
    Uq, _ = np.linalg.qr(rng.standard_normal((I1, I2)))
    Vq, _ = np.linalg.qr(rng.standard_normal((I2, I2)))
    sig = np.array([10.0, 7.0, 5.0, 1.0] + [0.5 / (k + 1) for k in range(I2 - 4)])
    Zm = (Uq * sig) @ Vq.T                   # I1 x I2 matrix
    dims = (I1, I2)
    Z = np.ascontiguousarray(Zm.T)           # numpy shape (I2, I1): mode 1 fastest
    A = [cpsynth.random_matrix(I1, R, 1), cpsynth.random_matrix(I2, R, 2)]
    for _ in range(60):
        A, out = oracle.als_sweep(Z, dims, A)
    s = np.linalg.svd(Zm, compute_uv=False)
    fstar = 0.5 * np.sum(s[R:] ** 2)
    assert out[0] == pytest.approx(fstar, rel=1e-10)
    assert oracle.f_direct(Z, dims, A) == pytest.approx(fstar, rel=1e-10)


def test_sweep_monotone_and_f_expand_matches_direct():
    """Each block update is an exact block minimizer so f is non-increasing
    (BJ); the sweep's expanded f equals the definition (eq:CPfunctional)."""
    d = cpsynth.make_config("c0", with_transfer=False)
    dims, Z, A = d["dims"], d["Z"], d["A0"]
    nz2 = float(np.vdot(Z, Z))
    prev = oracle.f_direct(Z, dims, A)
    for it in range(50):
        A, out = oracle.als_sweep(Z, dims, A, normZ2=nz2)
        assert out[2] == 0
        fd = oracle.f_direct(Z, dims, A)
        assert abs(out[0] - fd) <= 1e-10 * fd + 1e-14 * 0.5 * nz2
        assert fd <= prev * (1 + 1e-12)
        prev = fd


def test_sweep_with_rhs_monotone_ftilde():
    """f_tilde = f - sum_n <F^(n), A^(n)> is the functional whose block minimizers the
    BNGS-with-RHS update (eq:relaxinnersolve P:356-358) computes: non-increasing."""
    dims = (6, 5, 7)
    Z, A = cpsynth.random_problem(dims, 2, seed=77)
    # f_tilde is unbounded below along the scaling indeterminacy (the linear term wins), so
    # only a few sweeps with a small F are taken -- monotonicity holds at every step anyway.
    F = [0.05 * cpsynth.random_matrix(I, 2, seed=90 + k) for k, I in enumerate(dims)]
    prev = None
    for _ in range(8):
        A, out = oracle.als_sweep(Z, dims, A, F=F)
        ft = oracle.f_direct(Z, dims, A) - sum(np.vdot(f, a) for f, a in zip(F, A))
        assert out[1] == pytest.approx(ft, rel=1e-10, abs=1e-12)
        if prev is not None:
            assert ft <= prev + 1e-12 * abs(prev)
        prev = ft


def test_sweep_fixed_point_exact_solution():
    """The exact solution of a noiseless well-conditioned instance is unchanged."""
    dims = (9, 8, 7)
    Z, At, _ = cpsynth.lowrank_problem(dims, 3, seed=4, C=0.5)
    A1, out = oracle.als_sweep(Z, dims, At)
    for a, b in zip(A1, At):
        assert rel(a, b) <= 1e-12


def test_fas_fixed_point():
    """With F = H(A*) (eq:FASop), A* is a fixed point of BNGS with RHS."""
    dims = (5, 6, 4)
    Z, As = cpsynth.random_problem(dims, 3, seed=88)
    _, H = oracle.gradient(Z, dims, As)        # G = -Z_(n)Phi + A Gamma = H^(n)(A*)
    A1, out = oracle.als_sweep(Z, dims, As, F=H)
    for a, b in zip(A1, As):
        assert rel(a, b) <= 1e-12


def test_gradient_after_sweep_last_mode_zero():
    """G^(N) ~ 0 right after a sweep: mode N was just solved exactly (eq:relaxinnersolve)."""
    dims = (8, 7, 6)
    Z, A = cpsynth.random_problem(dims, 3, seed=99)
    A1, _ = oracle.als_sweep(Z, dims, A)
    out, G = oracle.gradient(Z, dims, A1)
    assert math.sqrt(out[2 + 2]) <= 1e-13 * np.linalg.norm(Z)
    assert out[2 + 0] > 1e-6


def test_singular_gamma_reported():
    """A zero factor column makes Gamma singular (Keller condition P:362): status ENOTSPD."""
    dims = (4, 5, 6)
    Z, A = cpsynth.random_problem(dims, 2, seed=5)
    A[2][:, 1] = 0.0
    _, out = oracle.als_sweep(Z, dims, A)
    assert out[2] == oracle.ENOTSPD and out[3] == 0


def test_recovery_noiseless_rank3():
    """Noiseless rank-3, C = 0.5, 20^3 (BJ): ALS + normalization reaches g < 1e-12 and the
    factors match the truth modulo scaling and permutation."""
    dims = (20, 20, 20)
    Z, At, A = cpsynth.lowrank_problem(dims, 3, seed=12, C=0.5)
    nz2 = float(np.vdot(Z, Z))
    g = 1.0
    for it in range(400):
        A, out = oracle.als_sweep(Z, dims, A, normZ2=nz2)
        A, lam = oracle.normalize_sort(dims, A)
        if it % 5 == 4:
            g = oracle.gradient(Z, dims, A, normZ2=nz2, want_G=False)[0][1]
            if g < 1e-12:
                break
    assert g < 1e-12
    for n in range(3):
        a = A[n] / np.linalg.norm(A[n], axis=0)
        t = At[n] / np.linalg.norm(At[n], axis=0)
        C = np.abs(a.T @ t)
        assert np.all(C.max(axis=1) > 1 - 1e-10)


def test_normalize_worked_example(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "normalize_example.json")))
    A = [np.asfortranarray(np.array(g["a"])[:, None]), np.asfortranarray(np.array(g["b"])[:, None])]
    An, lam = oracle.normalize_sort((2, 2), A)
    assert lam[0] == pytest.approx(g["lambda"], rel=1e-15)
    np.testing.assert_allclose(An[0][:, 0], g["a_out"], atol=1e-15)
    np.testing.assert_allclose(An[1][:, 0], g["b_out"], atol=1e-15)


def test_normalize_invariants():
    """eq:ALSnorm equilibrates column norms, keeps [[A]] unchanged, sorts lambda descending."""
    dims = (5, 6, 7)
    _, A = cpsynth.random_problem(dims, 4, seed=13)
    X0 = cpsynth.kruskal(A)
    An, lam = oracle.normalize_sort(dims, A)
    assert rel(cpsynth.kruskal(An), X0) <= 1e-13
    assert np.all(np.diff(lam) <= 0)
    for n in range(3):
        np.testing.assert_allclose(np.linalg.norm(An[n], axis=0), lam, rtol=1e-12)


def test_thread_count_independent():
    d = cpsynth.make_config("c0", with_transfer=False)
    res = []
    for t in (1, 3):
        oracle.set_threads(t)
        A, out = oracle.als_sweep(d["Z"], d["dims"], d["A0"])
        M = oracle.mttkrp(d["Z"], d["dims"], A, 1)
        res.append((A, out, M))
    oracle.set_threads(os.cpu_count() or 1)
    for a, b in zip(res[0][0], res[1][0]):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(res[0][1], res[1][1])
    np.testing.assert_array_equal(res[0][2], res[1][2])


# ---------------------------------------------------------------- mode products


def test_mode_product_identity_and_matrix_case():
    dims = (5, 4, 3)
    Z, _ = cpsynth.random_problem(dims, 1, seed=2)
    for n in range(3):
        X, nd = oracle.mode_product(Z, dims, n, np.eye(dims[n]))
        np.testing.assert_array_equal(X, Z)
    # order 2: X_(1) = U Z_(1) is a plain matrix product
    Zm = cpsynth.random_matrix(6, 9, 3)           # I1 x I2
    U = cpsynth.random_matrix(4, 6, 4)
    X, nd = oracle.mode_product(np.ascontiguousarray(Zm.T), (6, 9), 0, U)
    assert nd == [4, 9]
    np.testing.assert_allclose(X.T, U @ Zm, rtol=1e-13, atol=1e-13)
    V = cpsynth.random_matrix(2, 9, 5)
    X, nd = oracle.mode_product(np.ascontiguousarray(Zm.T), (6, 9), 1, V)
    np.testing.assert_allclose(X.T, Zm @ V.T, rtol=1e-13, atol=1e-13)


def test_mode_product_kronecker_identity_all_modes():
    """X = Z x_1 B1 ... x_N BN  <=>  X_(n) = B^(n) Z_(n) (B^(N) (x) .. (x) B^(1))^T without n
    (eq:propMatricized), on a 3x3x3x3 tensor; distinct modes commute."""
    dims = (3, 3, 3, 3)
    Z, _ = cpsynth.random_problem(dims, 1, seed=8)
    Bs = [cpsynth.random_matrix(J, 3, 20 + k) for k, J in enumerate((2, 3, 4, 1))]
    X, nd = Z, list(dims)
    for n in range(4):
        X, nd = oracle.mode_product(X, nd, n, Bs[n])
    for n in range(4):
        K = functools.reduce(np.kron, [Bs[k] for k in reversed(range(4)) if k != n])
        expect = Bs[n] @ unfold(Z, dims, n) @ K.T
        assert rel(unfold(X, nd, n), expect) <= 1e-13
    # commutation of distinct modes
    X1, d1 = oracle.mode_product(*oracle.mode_product(Z, dims, 0, Bs[0]), 2, Bs[2])
    X2, d2 = oracle.mode_product(*oracle.mode_product(Z, dims, 2, Bs[2]), 0, Bs[0])
    assert d1 == d2 and rel(X1, X2) <= 1e-14


def test_mode_product_kruskal_form_and_orthonormal_contraction():
    """[[A]] x_n U = [[..., U A^(n), ...]] (eq:propMatricized); an orthonormal-column Phat
    (Phat^T Phat = I) gives ||Z x_n Phat^T|| <= ||Z||."""
    dims = (8, 6, 7)
    _, A = cpsynth.random_problem(dims, 3, seed=14)
    Z = cpsynth.kruskal(A)
    U = cpsynth.random_matrix(4, 6, 15)
    X, nd = oracle.mode_product(Z, dims, 1, U)
    B = list(A)
    B[1] = U @ A[1]
    assert rel(X, cpsynth.kruskal(B)) <= 1e-13
    Zr, _ = cpsynth.random_problem(dims, 1, seed=16)
    Q, _ = np.linalg.qr(cpsynth.random_matrix(7, 4, 17))
    X, nd = oracle.mode_product(Zr, dims, 2, np.asfortranarray(Q.T))
    assert np.linalg.norm(X) <= np.linalg.norm(Zr) * (1 + 1e-15)


# ---------------------------------------------------------------- paper's dense problem


def test_dense_tensor_entry():
    """z_111 = 3^{-1/2} for the dense inverse-norm tensor."""
    assert cpsynth.dense_inverse_norm(3)[0, 0, 0] == pytest.approx(3 ** -0.5, rel=1e-16)


@pytest.mark.slow
def test_paper_dense_problem_als_converges(golden_dir):
    """Statistical smoke pin (Table 4 test 1): s = 50, R = 2, U(0,1) init, ALS with
    normalization reaches g < 1e-10 (eq:stopcrit).  Paper mean 161 iterations; we only
    require convergence within 10x that."""
    row = json.load(open(os.path.join(golden_dir, "table4_als.json")))["rows"][0]
    s, R = row["s"], row["R"]
    dims = (s, s, s)
    Z = cpsynth.dense_inverse_norm(s)
    nz2 = float(np.vdot(Z, Z))
    A = cpsynth.uniform_init(dims, R, seed=0)
    it_conv = None
    for it in range(1, 10 * row["als_it"] + 1):
        A, out = oracle.als_sweep(Z, dims, A, normZ2=nz2)
        A, _ = oracle.normalize_sort(dims, A)
        if it % 10 == 0:
            g = oracle.gradient(Z, dims, A, normZ2=nz2, want_G=False)[0][1]
            if g < 1e-10:
                it_conv = it
                break
    assert it_conv is not None
