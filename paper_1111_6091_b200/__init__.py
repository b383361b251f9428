"""paper_1111_6091_b200 -- B200 (sm_100a) hot path of the multigrid CP method of
De Sterck & Miller, arXiv 1111.6091: MTTKRP, the ALS / BNGS sweep with Cholesky solve and the
functional f, the n-mode products (restriction / interpolation) and f/g evaluation.

This module is a thin ctypes binding over ``lib/libcp.so`` (C ABI: ``include/cp.h``).  It only
marshals arguments: every arithmetic step runs in the library's CUDA kernels.  There is no CPU
fallback -- importing works without a GPU, but every call raises if the CUDA library or a CUDA
device is missing.

Tensor conventions:
  * Z: float64 CUDA tensor, contiguous, shape (I_N, ..., I_1)  (mode 1 fastest);
  * factor matrices A^(n), F^(n), G^(n) (I_n x R) and operators U (J x I_n): float64 CUDA
    tensors of that shape stored column-major, i.e. ``t.stride() == (1, rows)``; use
    :func:`colmajor` to convert.
  * modes are 0-based (mode 0 = the paper's mode 1).
"""
import ctypes
import os

import torch

from ._lib import (CP_ECUDA, CP_EDIM, CP_EINVAL, CP_ENOTSPD, CP_EWORKSPACE, CP_MAX_N, CP_MAX_R,
                   CP_OK, CPError, lib, lib_path)

__all__ = ["colmajor", "empty_factor", "Workspace", "norm2", "mttkrp", "als_sweep",
           "mode_product", "restrict_structured", "fit", "als_sweeps_then_gradient", "workspace_bytes", "lib", "lib_path", "last_launch_count",
           "CPError", "CP_OK", "CP_EINVAL", "CP_EDIM", "CP_ENOTSPD", "CP_ECUDA", "CP_EWORKSPACE"]


class _Shape(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("R", ctypes.c_int32), ("dims", ctypes.c_int64 * CP_MAX_N)]


def _shape(dims, R):
    s = _Shape()
    s.N = len(dims)
    s.R = int(R)
    for i, d in enumerate(dims):
        s.dims[i] = int(d)
    return s


def colmajor(t):
    """Column-major (Fortran-order) copy/view of a 2-D tensor: stride (1, rows)."""
    if t.dim() != 2:
        raise ValueError("expected a 2-D tensor")
    if t.stride(0) == 1 and (t.stride(1) == t.shape[0] or t.shape[1] == 1):
        return t
    return t.t().contiguous().t()


def empty_factor(rows, cols, device="cuda", dtype=torch.float64):
    return torch.empty((cols, rows), device=device, dtype=dtype).t()


def _check_cm(t, rows, cols, name):
    if t.dtype != torch.float64 or not t.is_cuda:
        raise TypeError(f"{name}: expected a float64 CUDA tensor")
    if tuple(t.shape) != (rows, cols):
        raise ValueError(f"{name}: expected shape {(rows, cols)}, got {tuple(t.shape)}")
    if rows > 1 and cols > 1 and not (t.stride(0) == 1 and t.stride(1) == rows):
        raise ValueError(f"{name}: must be column-major (use colmajor())")


def _check_Z(Z, dims):
    if Z.dtype != torch.float64 or not Z.is_cuda or not Z.is_contiguous():
        raise TypeError("Z: expected a contiguous float64 CUDA tensor")
    n = 1
    for d in dims:
        n *= int(d)
    if Z.numel() != n:
        raise ValueError(f"Z: {Z.numel()} elements, dims {tuple(dims)} need {n}")


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p()


def _ptr_array(ts):
    arr = (ctypes.c_void_p * len(ts))()
    for i, t in enumerate(ts):
        arr[i] = t.data_ptr() if t is not None else None
    return arr


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _check(code, what):
    if code != CP_OK:
        raise CPError(code, what)


def workspace_bytes(dims, R):
    lib()
    return int(lib().cp_workspace_bytes(ctypes.byref(_shape(dims, R))))


class Workspace:
    """Caller-owned device workspace (the library allocates nothing)."""

    def __init__(self, dims, R, device="cuda"):
        self.dims = tuple(int(d) for d in dims)
        self.R = int(R)
        self.nbytes = max(256, workspace_bytes(self.dims, self.R))
        self.buf = torch.empty(self.nbytes, dtype=torch.uint8, device=device)
        self._fits = {(self.dims, self.R): True}

    def fits(self, dims, R):
        key = (tuple(int(d) for d in dims), int(R))
        if key not in self._fits:
            self._fits[key] = workspace_bytes(*key) <= self.nbytes
        return self._fits[key]


def _ws(ws, dims, R, device):
    if ws is None:
        ws = Workspace(dims, R, device)
    elif not ws.fits(dims, R):
        raise CPError(CP_EWORKSPACE, "workspace too small")
    return ws


def last_launch_count():
    return int(lib().cp_last_launch_count())


def profile_enable(on=True):
    _check(lib().cp_profile_enable(1 if on else 0), "cp_profile_enable")


def profile_read():
    """(launches, total_ms, algorithmic_bytes) of the streaming-kernel launches since the last read."""
    n = ctypes.c_int64()
    ms = ctypes.c_double()
    b = ctypes.c_double()
    _check(lib().cp_profile_read(ctypes.byref(n), ctypes.byref(ms), ctypes.byref(b)), "cp_profile_read")
    return int(n.value), float(ms.value), float(b.value)


def norm2(Z, dims, out=None, ws=None, stream=None):
    """||Z||^2 as a 1-element float64 CUDA tensor (cp_norm2)."""
    _check_Z(Z, dims)
    out = torch.empty(1, dtype=torch.float64, device=Z.device) if out is None else out
    ws = _ws(ws, dims, 1, Z.device)
    _check(lib().cp_norm2(ctypes.byref(_shape(dims, 1)), _ptr(Z), _ptr(out), _ptr(ws.buf),
                          ctypes.c_size_t(ws.nbytes), _stream(stream)), "cp_norm2")
    return out


def mttkrp(Z, dims, A, mode, M=None, ws=None, stream=None):
    """M = Z_(mode) Phi^(mode)  (I_mode x R, column-major)   (cp_mttkrp)."""
    _check_Z(Z, dims)
    R = next(a for k, a in enumerate(A) if k != mode).shape[1]
    for k, a in enumerate(A):
        if k != mode:
            _check_cm(a, dims[k], R, f"A[{k}]")
    M = empty_factor(dims[mode], R, Z.device) if M is None else M
    _check_cm(M, dims[mode], R, "M")
    ws = _ws(ws, dims, R, Z.device)
    _check(lib().cp_mttkrp(ctypes.byref(_shape(dims, R)), _ptr(Z),
                           _ptr_array([a if k != mode else None for k, a in enumerate(A)]),
                           ctypes.c_int32(mode), _ptr(M), _ptr(ws.buf), ctypes.c_size_t(ws.nbytes),
                           _stream(stream)), "cp_mttkrp")
    return M


def als_sweep(Z, dims, A, normZ2, F=None, out=None, ws=None, stream=None, nsweeps=1, normalize=False):
    """nsweeps (default 1) ALS/BNGS sweeps, A updated in place; normalize=True follows every sweep
    by the eq:ALSnorm normalization without sorting (CP_SWEEPS_NORMALIZE).  Returns the device
    tensor out = [f, f_tilde, status, failed_mode] after the last sweep (cp_als_sweep /
    cp_als_sweeps)."""
    _check_Z(Z, dims)
    R = A[0].shape[1]
    for k, a in enumerate(A):
        _check_cm(a, dims[k], R, f"A[{k}]")
    Fp = None
    if F is not None:
        for k, f in enumerate(F):
            if f is not None:
                _check_cm(f, dims[k], R, f"F[{k}]")
        Fp = _ptr_array(list(F))
    out = torch.empty(4, dtype=torch.float64, device=Z.device) if out is None else out
    ws = _ws(ws, dims, R, Z.device)
    if nsweeps == 1 and not normalize:
        _check(lib().cp_als_sweep(ctypes.byref(_shape(dims, R)), _ptr(Z), _ptr(normZ2), _ptr_array(A),
                                  Fp, _ptr(out), _ptr(ws.buf), ctypes.c_size_t(ws.nbytes),
                                  _stream(stream)), "cp_als_sweep")
    else:
        _check(lib().cp_als_sweeps(ctypes.byref(_shape(dims, R)), _ptr(Z), _ptr(normZ2), _ptr_array(A),
                                   Fp, ctypes.c_int32(int(nsweeps)), ctypes.c_int32(1 if normalize else 0),
                                   _ptr(out), _ptr(ws.buf),
                                   ctypes.c_size_t(ws.nbytes), _stream(stream)), "cp_als_sweeps")
    return out


def mode_product(Z, dims, mode, U, X=None, stream=None):
    """X = Z x_mode U with U (J x I_mode, column-major).  Returns (X, new dims)."""
    _check_Z(Z, dims)
    J = U.shape[0]
    _check_cm(U, J, dims[mode], "U")
    nd = list(dims)
    nd[mode] = J
    if X is None:
        X = torch.empty(tuple(reversed(nd)), dtype=torch.float64, device=Z.device)
    _check_Z(X, nd)
    d = (ctypes.c_int64 * len(dims))(*[int(x) for x in dims])
    _check(lib().cp_mode_product(ctypes.c_int32(len(dims)), d, _ptr(Z), ctypes.c_int32(mode),
                                 _ptr(U), ctypes.c_int64(J), _ptr(X), ctypes.c_void_p(),
                                 ctypes.c_size_t(0), _stream(stream)), "cp_mode_product")
    return X, nd


def restrict_structured(Z, dims, mode, wl, wr, X=None, ws=None, stream=None):
    """X = Z x_mode Phat^T for the BAMG transfer operator of the geometric C/F splitting
    (cp_restrict_structured): C points 2j injected, F point 2j+1
    interpolated with weights wl[2j+1] (coarse j) and wr[2j+1] (coarse j+1); Phat = P L^{-T},
    P^T P = L L^T.  wl, wr: float64 CUDA vectors of length dims[mode].  Returns (X, new dims)."""
    _check_Z(Z, dims)
    I = int(dims[mode])
    for name, w in (("wl", wl), ("wr", wr)):
        if w.dtype != torch.float64 or not w.is_cuda or w.numel() != I or not w.is_contiguous():
            raise ValueError(f"{name}: expected a contiguous float64 CUDA vector of length {I}")
    nd = list(dims)
    nd[mode] = (I + 1) // 2
    if X is None:
        X = torch.empty(tuple(reversed(nd)), dtype=torch.float64, device=Z.device)
    _check_Z(X, nd)
    d = (ctypes.c_int64 * len(dims))(*[int(x) for x in dims])
    need = int(lib().cp_restrict_workspace_bytes(ctypes.c_int32(len(dims)), d, ctypes.c_int32(mode)))
    if ws is None or ws.numel() < need:
        ws = torch.empty(max(need, 32), dtype=torch.uint8, device=Z.device)
    _check(lib().cp_restrict_structured(ctypes.c_int32(len(dims)), d, _ptr(Z), ctypes.c_int32(mode),
                                        _ptr(wl), _ptr(wr), _ptr(X), _ptr(ws), ctypes.c_size_t(ws.numel()),
                                        _stream(stream)), "cp_restrict_structured")
    return X, nd


def normalize_sort(dims, A, sort=True, lam=None, ws=None, stream=None):
    """eq:ALSnorm normalization (+ decreasing-lambda ordering) of the factors, in place."""
    R = A[0].shape[1]
    for k, a in enumerate(A):
        _check_cm(a, dims[k], R, f"A[{k}]")
    ws = _ws(ws, dims, R, A[0].device)
    _check(lib().cp_normalize_sort(ctypes.byref(_shape(dims, R)), _ptr_array(A), ctypes.c_int32(1 if sort else 0),
                                   _ptr(lam), _ptr(ws.buf), ctypes.c_size_t(ws.nbytes), _stream(stream)),
           "cp_normalize_sort")
    return A


class MGParams(ctypes.Structure):
    """cp_mg_params (include/cp.h); defaults = Table 1 of the paper."""
    _fields_ = [("nu1_setup", ctypes.c_int32), ("nu2_setup", ctypes.c_int32), ("nuc_setup", ctypes.c_int32),
                ("n_test", ctypes.c_int32), ("nu1_solve", ctypes.c_int32), ("nu2_solve", ctypes.c_int32),
                ("nuc_solve", ctypes.c_int32), ("max_setup_cycles", ctypes.c_int32),
                ("min_setup_cycles", ctypes.c_int32), ("stagnation_eps", ctypes.c_double),
                ("use_fmg", ctypes.c_int32), ("nu_fmg", ctypes.c_int32), ("max_cycles", ctypes.c_int32),
                ("tol", ctypes.c_double), ("coarsest", ctypes.c_int32), ("solve_stagnation_after", ctypes.c_int32),
                ("max_trace", ctypes.c_int32), ("fmg_guard", ctypes.c_int32)]

    @classmethod
    def default(cls, **kw):
        p = cls()
        lib().cp_mg_default_params(ctypes.byref(p))
        for k, v in kw.items():
            setattr(p, k, v)
        return p


def mg_levels(dims, R, coarsest=0):
    """Level sizes of the hierarchy the driver builds (coarsen every mode with I_n > I_coarsest)."""
    c = coarsest if coarsest > 0 else 2 * R
    out = [tuple(int(d) for d in dims)]
    while any(d > c for d in out[-1]):
        out.append(tuple((d + 1) // 2 if d > c else d for d in out[-1]))
    return out


def mg_solve(Z, dims, A, T, A_fmg=None, params=None, stream=None):
    """Multigrid CP solve (cp_mg_solve).  A: boot factors (in/out); T: list of n_test lists of N
    test factor matrices; A_fmg: coarsest-level FMG initial guess (needed when use_fmg).
    Returns (report dict, trace array)."""
    import numpy as np
    _check_Z(Z, dims)
    N = len(dims)
    R = A[0].shape[1]
    params = params or MGParams.default()
    if params.max_trace <= 0:
        params.max_trace = 1024
    flatT = [t for block in T for t in block]
    if len(flatT) != params.n_test * N:
        raise ValueError("T must hold n_test blocks of N factor matrices")
    s = _shape(dims, R)
    nbytes = int(lib().cp_mg_workspace_bytes(ctypes.byref(s), ctypes.byref(params)))
    if nbytes == 0:
        raise CPError(CP_EINVAL, "cp_mg_workspace_bytes")
    buf = torch.empty(nbytes, dtype=torch.uint8, device=Z.device)
    report = (ctypes.c_double * 16)()
    trace = (ctypes.c_double * (4 * params.max_trace))()
    _check(lib().cp_mg_solve(ctypes.byref(s), _ptr(Z), _ptr_array(A), _ptr_array(flatT),
                             _ptr_array(A_fmg) if A_fmg is not None else None, ctypes.byref(params),
                             report, trace, _ptr(buf), ctypes.c_size_t(nbytes), _stream(stream)), "cp_mg_solve")
    keys = ["g", "f", "cycles", "setup_cycles", "solve_cycles", "levels", "status", "trace_rows", "rebuilds",
            "seconds", "fit_seconds", "failed_mode"]
    rep = {k: report[i] for i, k in enumerate(keys)}
    tr = np.array(trace[: 4 * int(rep["trace_rows"])]).reshape(-1, 4)
    return rep, tr


def als_solve(Z, dims, A, tol=1e-10, max_iters=10000, check_every=1, stream=None):
    """Standalone ALS with normalization until g < tol (cp_als_solve).  Returns a report dict."""
    _check_Z(Z, dims)
    R = A[0].shape[1]
    s = _shape(dims, R)
    nbytes = int(lib().cp_als_solve_workspace_bytes(ctypes.byref(s)))
    buf = torch.empty(nbytes, dtype=torch.uint8, device=Z.device)
    report = (ctypes.c_double * 8)()
    _check(lib().cp_als_solve(ctypes.byref(s), _ptr(Z), _ptr_array(A), ctypes.c_double(tol), ctypes.c_int32(max_iters),
                              ctypes.c_int32(check_every), report, _ptr(buf), ctypes.c_size_t(nbytes),
                              _stream(stream)), "cp_als_solve")
    keys = ["g", "f", "iterations", "status", "seconds", "fit_seconds", "failed_mode"]
    return {k: report[i] for i, k in enumerate(keys)}


def fit(Z, dims, A, normZ2, F=None, want_G=False, out=None, ws=None, stream=None):
    """f (direct), g and ||G^(n)||^2 at one iterate (cp_fit).  Returns (out, G list or None)."""
    _check_Z(Z, dims)
    N = len(dims)
    R = A[0].shape[1]
    for k, a in enumerate(A):
        _check_cm(a, dims[k], R, f"A[{k}]")
    Fp = None
    if F is not None:
        for k, f in enumerate(F):
            if f is not None:
                _check_cm(f, dims[k], R, f"F[{k}]")
        Fp = _ptr_array(list(F))
    G = [empty_factor(dims[k], R, Z.device) for k in range(N)] if want_G else None
    out = torch.empty(2 + N, dtype=torch.float64, device=Z.device) if out is None else out
    ws = _ws(ws, dims, R, Z.device)
    _check(lib().cp_fit(ctypes.byref(_shape(dims, R)), _ptr(Z), _ptr(normZ2), _ptr_array(A), Fp,
                        _ptr(out), _ptr_array(G) if G else None, _ptr(ws.buf),
                        ctypes.c_size_t(ws.nbytes), _stream(stream)), "cp_fit")
    return out, G


def als_sweeps_then_gradient(Z, dims, A, normZ2, F=None, gF=None, nsweeps=1, normalize=False, want_G=True,
                             ws=None, stream=None):
    """cp_als_sweeps followed by cp_gradient(F = gF) at the new iterate in one call
    (cp_als_sweeps_then_gradient; one launch on small tensors).  Returns (out, gout, G list or None)."""
    _check_Z(Z, dims)
    N = len(dims)
    R = A[0].shape[1]
    for k, a in enumerate(A):
        _check_cm(a, dims[k], R, f"A[{k}]")

    def parr(Fs):
        if Fs is None:
            return None
        for k, f in enumerate(Fs):
            if f is not None:
                _check_cm(f, dims[k], R, f"F[{k}]")
        return _ptr_array(list(Fs))

    G = [empty_factor(dims[k], R, Z.device) for k in range(N)] if want_G else None
    out = torch.empty(4, dtype=torch.float64, device=Z.device)
    gout = torch.empty(2 + N, dtype=torch.float64, device=Z.device)
    ws = _ws(ws, dims, R, Z.device)
    _check(lib().cp_als_sweeps_then_gradient(
        ctypes.byref(_shape(dims, R)), _ptr(Z), _ptr(normZ2), _ptr_array(A), parr(F), ctypes.c_int32(int(nsweeps)),
        ctypes.c_int32(1 if normalize else 0), _ptr(out), parr(gF), _ptr(gout), _ptr_array(G) if G else None,
        _ptr(ws.buf), ctypes.c_size_t(ws.nbytes), _stream(stream)), "cp_als_sweeps_then_gradient")
    return out, gout, G


def gradient(Z, dims, A, normZ2, F=None, want_G=False, out=None, ws=None, stream=None):
    """g, ||G^(n)||^2 (and G) at one iterate without the residual pass, f by the expansion
    (cp_gradient).  Returns (out, G list or None)."""
    _check_Z(Z, dims)
    N = len(dims)
    R = A[0].shape[1]
    for k, a in enumerate(A):
        _check_cm(a, dims[k], R, f"A[{k}]")
    Fp = None
    if F is not None:
        for k, f in enumerate(F):
            if f is not None:
                _check_cm(f, dims[k], R, f"F[{k}]")
        Fp = _ptr_array(list(F))
    G = [empty_factor(dims[k], R, Z.device) for k in range(N)] if want_G else None
    out = torch.empty(2 + N, dtype=torch.float64, device=Z.device) if out is None else out
    ws = _ws(ws, dims, R, Z.device)
    _check(lib().cp_gradient(ctypes.byref(_shape(dims, R)), _ptr(Z), _ptr(normZ2), _ptr_array(A), Fp,
                             _ptr(out), _ptr_array(G) if G else None, _ptr(ws.buf),
                             ctypes.c_size_t(ws.nbytes), _stream(stream)), "cp_gradient")
    return out, G
