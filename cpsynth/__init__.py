"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds random-number recipes only -- none of the method's arithmetic (no MTTKRP,
no Gram/Cholesky solve, no mode product, no functional).  It serves both the oracle and the
CUDA path; neither of them imports the other.  The one non-random step, forming the
noiseless target T = [[A*]] of BASELINE.json's configs, is done with numpy library
primitives (a Khatri-Rao build and one dgemm) so that it is independent of both sides.

Layout: a dense tensor of size I_1 x ... x I_N is a C-contiguous
numpy array of shape (I_N, ..., I_1) -- mode 1 fastest, Kolda-Bader order -- and every
factor matrix is an I_n x R Fortran-order (column-major) float64 array.

Config recipe (BASELINE.json `configs`):
  ss = SeedSequence([11116091, c]); q, n1, n2, init, pop = [default_rng(s) for s in ss.spawn(5)]
  K = C*11^T + (1-C)I,  L = cholesky(K) (lower),  A*^(n) = qr(q.standard_normal((I_n,R)))[0] @ L^T
  T = [[A*]],  Z = T + l1*||T||/||N1||*N1 (+ l2*||T||/||N2*T||*(N2*T))
  A0^(n) = init.standard_normal((I_n, R))              (BASELINE.json: seeded N(0,1) guess)
  Phat^(n) = qr(pop.standard_normal((I_n, ceil(I_n/2))))[0]   (orthonormal columns, like the
            paper's Phat = P L^{-T}; restriction operator U = Phat^T)
"""
import math

import numpy as np

SEED_BASE = 11116091

# name: (index, dims, R, C, l1, l2, note)
CONFIGS = {
    "c0": (0, (20, 20, 20), 3, 0.5, 0.01, 0.0, "3-way 20^3 R=3 C=0.5 l1=1% (BASELINE.json configs[0])"),
    "c1": (1, (50, 50, 50), 3, 0.9, 0.01, 0.01, "3-way 50^3 R=3 C=0.9 l1=l2=1% (configs[1])"),
    "c2": (2, (100, 100, 100), 5, 0.9, 0.01, 0.01, "3-way 100^3 R=5 C=0.9 l1=l2=1% (configs[2])"),
    "c3": (3, (256, 256, 256), 8, 0.5, 0.01, 0.0, "3-way 256^3 R=8 C=0.5 l1=1% (configs[3])"),
    "c4a": (4, (512, 512, 512), 16, 0.9, 0.01, 0.01, "3-way 512^3 R=16 C=0.9 l1=l2=1% (configs[4])"),
    "c4b": (5, (96, 96, 96, 96), 10, 0.5, 0.01, 0.0, "4-way 96^4 R=10 C=0.5 l1=1% (configs[4])"),
}


def tensor_shape(dims):
    """numpy shape of a tensor with sizes dims = (I_1..I_N): (I_N, ..., I_1)."""
    return tuple(reversed([int(d) for d in dims]))


def khatri_rao_rows(mats):
    """Rows of mats[-1] (.) ... (.) mats[0] with mats[0]'s index fastest (Kolda order)."""
    R = mats[0].shape[1]
    phi = np.ascontiguousarray(mats[0])
    for m in mats[1:]:
        phi = np.einsum("jr,kr->kjr", phi, m).reshape(-1, R)
    return phi


def kruskal(A):
    """Dense T = [[A^(1), ..., A^(N)]] (numpy library primitives; input recipe only)."""
    dims = [a.shape[0] for a in A]
    if len(A) == 1:
        return A[0].sum(axis=1)
    phi = khatri_rao_rows(A[1:])                  # (prod_{k>1} I_k) x R
    T = phi @ np.ascontiguousarray(A[0]).T        # [j, i1] -> i1 fastest
    return np.ascontiguousarray(T).reshape(tensor_shape(dims))


def congruence_factors(rng, dims, R, C):
    K = C * np.ones((R, R)) + (1.0 - C) * np.eye(R)
    L = np.linalg.cholesky(K)  # lower, K = L L^T  (SURVEY 8(c) reading 10)
    out = []
    for I in dims:
        Q, _ = np.linalg.qr(rng.standard_normal((I, R)))
        out.append(np.asfortranarray(Q @ L.T))
    return out


def make_config(name, with_transfer=True):
    """Build BASELINE.json config `name`.  Returns a dict of numpy arrays (see module doc)."""
    c, dims, R, C, l1, l2, note = CONFIGS[name]
    ss = np.random.SeedSequence([SEED_BASE, c])
    rq, rn1, rn2, rinit, rpop = [np.random.default_rng(s) for s in ss.spawn(5)]
    A_true = congruence_factors(rq, dims, R, C)
    T = kruskal(A_true)
    nT = math.sqrt(float(np.vdot(T, T)))
    Z = T.copy()
    N1 = rn1.standard_normal(T.shape)
    Z += (l1 * nT / math.sqrt(float(np.vdot(N1, N1)))) * N1
    del N1
    if l2 > 0:
        W = rn2.standard_normal(T.shape)
        W *= T
        Z += (l2 * nT / math.sqrt(float(np.vdot(W, W)))) * W
        del W
    del T
    A0 = [np.asfortranarray(rinit.standard_normal((I, R))) for I in dims]
    out = dict(name=name, dims=tuple(dims), R=R, C=C, l1=l1, l2=l2, note=note, Z=Z,
               A_true=A_true, A0=A0, normT=nT)
    if with_transfer:
        Ph = []
        for I in dims:
            Ic = (I + 1) // 2
            Q, _ = np.linalg.qr(rpop.standard_normal((I, Ic)))
            Ph.append(np.asfortranarray(Q))
        out["Phat"] = Ph
    return out


def random_problem(dims, R, seed, scale_A=1.0):
    """Gaussian Z and N(0,1) factors for parity tests on arbitrary (ragged) shapes."""
    rng = np.random.default_rng(np.random.SeedSequence([SEED_BASE, 1000, seed]))
    Z = rng.standard_normal(tensor_shape(dims))
    A = [np.asfortranarray(scale_A * rng.standard_normal((I, R))) for I in dims]
    return Z, A


def transfer_weights(I, seed):
    """F-row interpolation weights (wl, wr) in [0.2, 0.8] -- the range of the least-squares
    weights of the paper's smooth problems (linear vectors give exactly 1/2) -- for
    the structured restriction (cp_restrict_structured / oracle.mg.restrict_structured)."""
    rng = np.random.default_rng(np.random.SeedSequence([SEED_BASE, 3000, seed]))
    return rng.uniform(0.2, 0.8, I), rng.uniform(0.2, 0.8, I)


def random_matrix(rows, cols, seed):
    rng = np.random.default_rng(np.random.SeedSequence([SEED_BASE, 2000, seed]))
    return np.asfortranarray(rng.standard_normal((rows, cols)))


def lowrank_problem(dims, R, seed, C=0.5, noise=0.0):
    """Z = [[A*]] (+ relative Gaussian noise) with congruence-C factors; returns (Z, A_true, A0)."""
    ss = np.random.SeedSequence([SEED_BASE, 3000, seed])
    rq, rn, rinit = [np.random.default_rng(s) for s in ss.spawn(3)]
    A_true = congruence_factors(rq, dims, R, C)
    Z = kruskal(A_true)
    if noise > 0:
        N1 = rn.standard_normal(Z.shape)
        Z = Z + noise * np.linalg.norm(Z) / np.linalg.norm(N1) * N1
    A0 = [np.asfortranarray(rinit.standard_normal((I, R))) for I in dims]
    return Z, A_true, A0


def dense_inverse_norm(s):
    """The paper's dense test tensor z_ijk = (i^2+j^2+k^2)^{-1/2}, i,j,k = 1..s."""
    i = np.arange(1, s + 1, dtype=np.float64)
    return 1.0 / np.sqrt(i[:, None, None] ** 2 + i[None, :, None] ** 2 + i[None, None, :] ** 2)


def uniform_init(dims, R, seed):
    """Standard-uniform initial guesses as in the paper's experiments."""
    rng = np.random.default_rng(np.random.SeedSequence([SEED_BASE, 4000, seed]))
    return [np.asfortranarray(rng.uniform(size=(I, R))) for I in dims]
