"""ctypes wrapper around liboracle.so -- the plain CPU fp64 ORACLE (see cp_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this module.
The product path (``paper_1111_6091_b200``) never imports it and shares no code with it.

Every function takes/returns numpy float64 arrays in the layout of DESIGN.md:
  * a dense tensor of size I_1 x ... x I_N is a contiguous numpy array of shape
    (I_N, ..., I_1) (mode 1 fastest) -- equivalently ``Z.reshape(-1)`` is the
    Kolda-order vector;
  * factor matrices / M / F / G / U are 2-D numpy arrays in Fortran order (column-major).
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int64_p = ctypes.POINTER(ctypes.c_int64)

ENOTSPD = -3


def build(verbose=False):
    """Compile liboracle.so with gcc (plain C11, -O2, OpenMP, no fast-math)."""
    import subprocess
    src = os.path.join(_HERE, "cp_oracle.c")
    cmd = ["gcc", "-std=c11", "-O2", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
           "-ffp-contract=off", "-o", _LIB_PATH, src, "-lm"]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "cp_oracle.c"))):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_norm2.restype = ctypes.c_double
        L.oracle_f_direct.restype = ctypes.c_double
        I, I64, D, DP, LP = ctypes.c_int, ctypes.c_int64, ctypes.c_double, c_double_p, c_int64_p
        PP = ctypes.POINTER(c_double_p)
        L.oracle_norm2.argtypes = [I, LP, DP]
        L.oracle_mttkrp_rows.argtypes = [I, LP, I, DP, PP, I, I64, I64, DP]
        L.oracle_mttkrp.argtypes = [I, LP, I, DP, PP, I, DP]
        L.oracle_gram.argtypes = [I64, I, DP, DP]
        L.oracle_gamma.argtypes = [I, I, PP, I, DP]
        L.oracle_cholesky.argtypes = [I, DP, DP]
        L.oracle_solve_rows.argtypes = [I64, I, DP, DP, DP]
        L.oracle_als_sweep.argtypes = [I, LP, I, DP, D, PP, PP, DP]
        L.oracle_f_direct.argtypes = [I, LP, I, DP, PP]
        L.oracle_gradient.argtypes = [I, LP, I, DP, D, PP, PP, DP, PP]
        L.oracle_mode_product.argtypes = [I, LP, DP, I, DP, I64, DP]
        L.oracle_normalize_sort.argtypes = [I, LP, I, PP, DP]
        L.oracle_normalize.argtypes = [I, LP, I, PP, DP, I]
        L.oracle_normalize.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [I]
        L.oracle_set_threads.restype = None
        for name in ["oracle_mttkrp_rows", "oracle_mttkrp", "oracle_gram", "oracle_gamma",
                     "oracle_cholesky", "oracle_solve_rows", "oracle_als_sweep",
                     "oracle_gradient", "oracle_mode_product", "oracle_normalize_sort",
                     "oracle_num_threads"]:
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(c_double_p)


def _dims(dims):
    arr = (ctypes.c_int64 * len(dims))(*[int(d) for d in dims])
    return arr


def _ptr_array(mats):
    arr = (c_double_p * len(mats))()
    for i, m in enumerate(mats):
        arr[i] = _dp(m) if m is not None else c_double_p()
    return arr


def _cm(a):
    a = np.asarray(a, dtype=np.float64)
    return np.asfortranarray(a)


def _zvec(Z, dims):
    Z = np.ascontiguousarray(Z, dtype=np.float64)
    assert Z.size == int(np.prod(dims)), (Z.shape, dims)
    return Z.reshape(-1)


def num_threads():
    return lib().oracle_num_threads()


def set_threads(n):
    lib().oracle_set_threads(int(n))


def norm2(Z):
    Z = np.ascontiguousarray(Z, dtype=np.float64).reshape(-1)
    dims = [Z.size]
    return lib().oracle_norm2(1, _dims(dims), _dp(Z))


def mttkrp(Z, dims, A, mode, rows=None):
    """M = Z_(mode) Phi^(mode), I_mode x R (Fortran order). rows=(lo,hi) fills only those rows."""
    N = len(dims)
    R = A[0].shape[1]
    z = _zvec(Z, dims)
    A = [_cm(a) for a in A]
    M = np.zeros((dims[mode], R), dtype=np.float64, order="F")
    lo, hi = (0, dims[mode]) if rows is None else rows
    st = lib().oracle_mttkrp_rows(N, _dims(dims), R, _dp(z), _ptr_array(A), mode, lo, hi, _dp(M))
    if st != 0:
        raise ValueError(f"oracle_mttkrp_rows status {st}")
    return M


def gram(A):
    A = _cm(A)
    R = A.shape[1]
    U = np.zeros((R, R), order="F")
    lib().oracle_gram(A.shape[0], R, _dp(A), _dp(U))
    return U


def cholesky(G):
    G = _cm(G)
    R = G.shape[0]
    L = np.zeros((R, R), order="F")
    st = lib().oracle_cholesky(R, _dp(G), _dp(L))
    return st, L


def solve_rows(L, B):
    L = _cm(L)
    B = _cm(B)
    X = np.zeros_like(B, order="F")
    lib().oracle_solve_rows(B.shape[0], B.shape[1], _dp(L), _dp(B), _dp(X))
    return X


def als_sweep(Z, dims, A, F=None, normZ2=None):
    """One ALS/BNGS sweep.  Returns (A_new list, out[4] = f, f_tilde, status, failed_mode)."""
    N = len(dims)
    R = A[0].shape[1]
    z = _zvec(Z, dims)
    if normZ2 is None:
        normZ2 = float(np.dot(z, z))
    A = [np.array(_cm(a), order="F", copy=True) for a in A]
    Fp = None
    if F is not None:
        F = [(_cm(f) if f is not None else None) for f in F]
        Fp = _ptr_array(F)
    out = np.zeros(4)
    st = lib().oracle_als_sweep(N, _dims(dims), R, _dp(z), ctypes.c_double(normZ2),
                                _ptr_array(A), Fp, _dp(out))
    if st != 0:
        raise ValueError(f"oracle_als_sweep status {st}")
    return A, out


def f_direct(Z, dims, A):
    z = _zvec(Z, dims)
    A = [_cm(a) for a in A]
    return lib().oracle_f_direct(len(dims), _dims(dims), A[0].shape[1], _dp(z), _ptr_array(A))


def f_expand(Z, dims, A, normZ2=None):
    """f at one iterate by the expansion (reading R6; eq:CPfunctional with eq:propMatricized and
    eq:Gamma P:113-116):  f = 1/2 ||Z||^2 - <Z_(N) Phi^(N), A^(N)> + 1/2 1^T (*_k A^(k)T A^(k)) 1,
    written from oracle_mttkrp and oracle_gram.  Pinned against f_direct (the plain definition),
    the exact-model and zero-factor special cases in tests/test_oracle_pins.py."""
    N = len(dims)
    z = _zvec(Z, dims)
    if normZ2 is None:
        normZ2 = float(np.dot(z, z))
    M = mttkrp(Z, dims, A, N - 1)
    inner = float(np.sum(M * _cm(A[N - 1])))
    H = np.ones((A[0].shape[1],) * 2)
    for a in A:
        H = H * gram(a)
    return 0.5 * normZ2 - inner + 0.5 * float(np.sum(H))


def gradient(Z, dims, A, F=None, normZ2=None, want_G=True):
    """Returns (out[2+N] = f, g, ||G^n||^2..., G list or None)."""
    N = len(dims)
    R = A[0].shape[1]
    z = _zvec(Z, dims)
    if normZ2 is None:
        normZ2 = float(np.dot(z, z))
    A = [_cm(a) for a in A]
    Fp = None
    if F is not None:
        F = [(_cm(f) if f is not None else None) for f in F]
        Fp = _ptr_array(F)
    out = np.zeros(2 + N)
    G = [np.zeros((dims[n], R), order="F") for n in range(N)] if want_G else None
    st = lib().oracle_gradient(N, _dims(dims), R, _dp(z), ctypes.c_double(normZ2), _ptr_array(A),
                               Fp, _dp(out), _ptr_array(G) if want_G else None)
    if st != 0:
        raise ValueError(f"oracle_gradient status {st}")
    return out, G


def mode_product(Z, dims, mode, U):
    """X = Z x_mode U with U (J x I_mode).  Returns (X as C-order array of shape reversed(new dims), new dims)."""
    N = len(dims)
    U = _cm(U)
    J = U.shape[0]
    assert U.shape[1] == dims[mode]
    z = _zvec(Z, dims)
    nd = list(dims)
    nd[mode] = J
    X = np.zeros(int(np.prod(nd)), dtype=np.float64)
    st = lib().oracle_mode_product(N, _dims(dims), _dp(z), mode, _dp(U), J, _dp(X))
    if st != 0:
        raise ValueError(f"oracle_mode_product status {st}")
    return X.reshape(list(reversed(nd))), nd


def normalize_sort(dims, A, sort=True):
    """eq:ALSnorm normalization; sort=True also orders the components by decreasing lambda."""
    N = len(dims)
    R = A[0].shape[1]
    A = [np.array(_cm(a), order="F", copy=True) for a in A]
    lam = np.zeros(R)
    lib().oracle_normalize(N, _dims(dims), R, _ptr_array(A), _dp(lam), 1 if sort else 0)
    return A, lam
