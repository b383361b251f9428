"""Plain CPU oracle of the multigrid CP method (De Sterck & Miller, arXiv 1111.6091), written
step by step from the paper -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Algorithms: CP-AMG-mult (Algorithm 1), CP-FAS (Algorithm 2),
FMG-CP-FAS (Algorithm 3) and the setup/solve combination of P:486-492, with the
DESIGN.md readings (R16 coarsest size 2R, R17 one-sided right end, R22 setup relaxations
normalize on every level, R23 FAS relaxations normalize + sort on the finest level only, R24
F_c = H_c(A~_c) + (F - H(A)) for uncoarsened modes).  Level work uses the C oracle
(oracle_als_sweep, oracle_gradient, oracle_mode_product, oracle_normalize); the transfer
operators use dense numpy/scipy linear algebra (P, B = P^T P, B = L L^T, Phat = P L^{-T}).
It shares no code with paper_1111_6091_b200.
"""
import numpy as np
from scipy.linalg import solve_triangular

import oracle


def levels(dims, R, coarsest=0):
    """Level sizes: coarsen mode n while I_n > I_coarsest, C = odd points."""
    c = coarsest if coarsest > 0 else 2 * R
    out = [tuple(int(d) for d in dims)]
    while any(d > c for d in out[-1]):
        out.append(tuple((d + 1) // 2 if d > c else d for d in out[-1]))
    return out


def interpolation_matrix(U_list, weights):
    """P of one mode: C points 0, 2, 4, ... (0-based; the paper's odd points) map to
    coarse point i/2 with weight 1; F point i interpolates from coarse (i-1)/2 and (i+1)/2
    (one-sided at an even right end).  The weights of each F row solve the weighted LS problem
    eq:LSQinterp by the normal equations, each fitted vector u_k (a column of U_list[t]) with the
    weight of its factor matrix (eq:interpweights)."""
    I = U_list[0].shape[0]
    Ic = (I + 1) // 2
    P = np.zeros((I, Ic))
    cols = np.concatenate(U_list, axis=1)                     # I x n_f
    w = np.concatenate([np.full(u.shape[1], wt) for u, wt in zip(U_list, weights)])
    for i in range(I):
        if i % 2 == 0:
            P[i, i // 2] = 1.0
            continue
        nb = [(i - 1) // 2] + ([(i + 1) // 2] if i + 1 < I else [])
        X = np.stack([cols[2 * j] for j in nb], axis=1)      # n_f x |C^i| (injection u_{k,c})
        y = cols[i]
        Aeq = X.T @ (w[:, None] * X)
        beq = X.T @ (w * y)
        P[i, nb] = np.linalg.solve(Aeq, beq)
    return P


def interpolation_from_weights(I, wl, wr):
    """P (I x ceil(I/2)) of the geometric C/F splitting with given F-row weights:
    P[2j, j] = 1; F point i = 2j+1: P[i, j] = wl[i], P[i, j+1] = wr[i] (one-sided at an even
    right end, reading R17) -- the sparsity pattern interpolation_matrix() fills by LS."""
    Ic = (I + 1) // 2
    P = np.zeros((I, Ic))
    for i in range(I):
        if i % 2 == 0:
            P[i, i // 2] = 1.0
        else:
            P[i, (i - 1) // 2] = wl[i]
            if i + 1 < I:
                P[i, (i + 1) // 2] = wr[i]
    return P


def restrict_structured(Z, dims, mode, wl, wr):
    """X = Z x_mode Phat^T with Phat from P (interpolation_from_weights) by transfer(): the
    definition of eq:ctensor_transformed, dense.  Returns (X, new dims)."""
    Ph = transfer(interpolation_from_weights(int(dims[mode]), wl, wr))
    return oracle.mode_product(Z, dims, mode, np.asfortranarray(Ph.T))


def transfer(P):
    """B = P^T P = L L^T, Phat = P L^{-T}, R = Phat^T."""
    B = P.T @ P
    L = np.linalg.cholesky(B)
    Ph = solve_triangular(L, P.T, lower=True).T
    return np.asfortranarray(Ph)


class Level:
    def __init__(self, dims, R, has_next, coarsest):
        self.dims = dims
        self.R = R
        self.has_next = has_next
        self.coarsen = [d > coarsest for d in dims] if has_next else [False] * len(dims)
        self.Z = None
        self.nz2 = None
        self.A = None
        self.T = None
        self.Ph = [None] * len(dims)


class MGOracle:
    def __init__(self, Z, dims, R, params):
        self.p = dict(params)
        self.N = len(dims)
        self.R = R
        c = self.p["coarsest"] if self.p["coarsest"] > 0 else 2 * R
        sizes = levels(dims, R, self.p["coarsest"])
        self.lv = [Level(d, R, k + 1 < len(sizes), c) for k, d in enumerate(sizes)]
        self.lv[0].Z = np.ascontiguousarray(Z, dtype=np.float64)
        self.lv[0].nz2 = float(np.vdot(Z, Z))
        self.fail = None  # failing mode of the first relaxation that hit a non-positive pivot

    def _note(self, out):
        """A relaxation reported CP_ENOTSPD (out[2] = -3): remember its mode.  The solve stops at
        the next stopping test with status -3 (Gamma singular: the Keller condition of P:362
        fails; the factors are then unspecified), as cp_mg_solve does."""
        if out[2] != 0 and self.fail is None:
            self.fail = int(out[3])

    # ---- building blocks
    def relax_setup(self, l, A, sweeps):
        v = self.lv[l]
        for _ in range(sweeps):
            A, out = oracle.als_sweep(v.Z, v.dims, A, normZ2=v.nz2)
            self._note(out)
            A, _ = oracle.normalize_sort(v.dims, A, sort=False)
        return A

    def relax_fas(self, l, A, F, sweeps):
        v = self.lv[l]
        for _ in range(sweeps):
            A, out = oracle.als_sweep(v.Z, v.dims, A, F=F, normZ2=v.nz2)
            self._note(out)
            if l == 0:
                A, _ = oracle.normalize_sort(v.dims, A, sort=True)
        return A

    def fit(self, l, A, want_G=False):
        v = self.lv[l]
        out, G = oracle.gradient(v.Z, v.dims, A, normZ2=v.nz2, want_G=want_G)
        return out, G

    def restrict(self, l, X):
        v = self.lv[l]
        return [np.asfortranarray(v.Ph[n].T @ X[n]) if v.coarsen[n] else X[n].copy(order="F")
                for n in range(self.N)]

    def interp(self, l, X):
        v = self.lv[l]
        return [np.asfortranarray(v.Ph[n] @ X[n]) if v.coarsen[n] else X[n].copy(order="F")
                for n in range(self.N)]

    def build_ops(self, l, first):
        v = self.lv[l]
        nt = len(v.T)
        gn = [self.fit(l, v.T[t])[0][2:] for t in range(nt)]
        if not first:
            gn.append(self.fit(l, v.A)[0][2:])
        for n in range(self.N):
            if not v.coarsen[n]:
                continue
            U = [v.T[t][n] for t in range(nt)] + ([] if first else [v.A[n]])
            wts = [float(np.sum(U[t] ** 2)) / gn[t][n] for t in range(len(U))]
            v.Ph[n] = transfer(interpolation_matrix(U, wts))
        nx = self.lv[l + 1]
        Zc, d = v.Z, list(v.dims)
        for n in range(self.N):
            if v.coarsen[n]:
                Zc, d = oracle.mode_product(Zc, d, n, np.asfortranarray(v.Ph[n].T))
        nx.Z = Zc
        nx.nz2 = float(np.vdot(Zc, Zc))

    # ---- Algorithm 1
    def setup_cycle(self, l, first, update_boot):
        v = self.lv[l]
        if not v.has_next:
            if update_boot:
                v.A = self.relax_setup(l, v.A, self.p["nuc_setup"])
            return
        v.T = [self.relax_setup(l, T, self.p["nu1_setup"]) for T in v.T]
        if update_boot:
            v.A = self.relax_setup(l, v.A, self.p["nu1_setup"])
        self.build_ops(l, first)
        nx = self.lv[l + 1]
        nx.A = self.restrict(l, v.A)
        nx.T = [self.restrict(l, T) for T in v.T]
        self.setup_cycle(l + 1, first, update_boot)
        if update_boot:
            v.A = self.interp(l, nx.A)
            v.A = self.relax_setup(l, v.A, self.p["nu2_setup"])

    # ---- Algorithm 2
    def fas_cycle(self, l, F):
        v = self.lv[l]
        if not v.has_next:
            v.A = self.relax_fas(l, v.A, F, self.p["nuc_solve"])
            return
        v.A = self.relax_fas(l, v.A, F, self.p["nu1_solve"])
        nx = self.lv[l + 1]
        Atil = self.restrict(l, v.A)
        _, H = self.fit(l, v.A, want_G=True)
        _, Hc = self.fit(l + 1, Atil, want_G=True)
        resid = [(-H[n] if F is None else F[n] - H[n]) for n in range(self.N)]
        rr = self.restrict(l, resid)
        Fc = [np.asfortranarray(Hc[n] + rr[n]) for n in range(self.N)]
        nx.A = [a.copy(order="F") for a in Atil]
        self.fas_cycle(l + 1, Fc)
        corr = self.interp(l, [nx.A[n] - Atil[n] for n in range(self.N)])
        v.A = [np.asfortranarray(v.A[n] + corr[n]) for n in range(self.N)]
        v.A = self.relax_fas(l, v.A, F, self.p["nu2_solve"])

    # ---- Algorithm 3
    def fmg(self, A_fmg):
        L = len(self.lv)
        c = self.lv[L - 1]
        c.A = self.relax_setup(L - 1, [a.copy(order="F") for a in A_fmg], self.p["nu_fmg"])
        for l in range(L - 1, 0, -1):
            self.lv[l - 1].A = self.interp(l - 1, self.lv[l].A)
            self.fas_cycle(l - 1, None)

    def stop_g(self):
        """g at the finest level for a stopping test; NaN once a relaxation has failed."""
        return float("nan") if self.fail is not None else self.fit(0, self.lv[0].A)[0][1]

    # ---- combination
    def solve(self, A0, T0, A_fmg=None):
        p = self.p
        f = self.lv[0]
        f.A = [np.asfortranarray(a) for a in A0]
        f.T = [[np.asfortranarray(t) for t in blk] for blk in T0]
        trace = []
        g = self.fit(0, f.A)[0][1]
        converged = g < p["tol"]
        cycles = setup_cycles = solve_cycles = rebuilds = 0
        g_old = g
        for cyc in range(1, p["max_setup_cycles"] + 1):
            if converged:
                break
            self.setup_cycle(0, cyc == 1, True)
            gn = self.stop_g()
            cycles += 1
            setup_cycles += 1
            trace.append((0, cycles, gn))
            g = gn
            if not gn >= p["tol"]:
                converged = (gn == gn) and gn < p["tol"]
                break
            if cyc >= p["min_setup_cycles"] and gn > (1.0 - p["stagnation_eps"]) * g_old:
                break
            g_old = gn
        if not converged and p["use_fmg"] and self.fail is None:
            # "Multilevel + FMG": one FMG-CP-FAS cycle computes a new approximation to the
            # boot factors, then the transfer operators are rebuilt by one down-sweep of
            # CP-AMG-mult (boot factors not updated).  fmg_guard = 1 is reading R29 (not the
            # paper's default): the FMG result is kept only if it lowers g, else the setup
            # iterate is restored and the operators are not rebuilt.
            kept = [a.copy(order="F") for a in f.A]
            self.fmg(A_fmg)
            gf = self.stop_g()
            cycles += 1
            trace.append((1, cycles, gf))
            if p["fmg_guard"] and not gf < g:
                f.A = kept
            else:
                g = gf
                converged = g < p["tol"]
                if not converged and self.fail is None:
                    self.setup_cycle(0, False, False)
        rebuilt = False
        g_old = g
        while not converged and cycles < p["max_cycles"] and self.fail is None:
            prev = [a.copy(order="F") for a in f.A]
            self.fas_cycle(0, None)
            gn = self.stop_g()
            cycles += 1
            solve_cycles += 1
            trace.append((2, cycles, gn))
            if gn != gn:
                break
            if gn < p["tol"]:
                g = gn
                converged = True
                break
            if solve_cycles > p["solve_stagnation_after"] and gn >= g_old and not rebuilt:
                f.A = prev
                self.setup_cycle(0, False, False)
                rebuilt = True
                rebuilds += 1
                gn = g_old
            g = gn
            g_old = gn
        out = self.fit(0, f.A)[0]
        status = -3 if self.fail is not None else (0 if converged else 1)
        report = dict(g=g, f=out[0], cycles=cycles, setup_cycles=setup_cycles, solve_cycles=solve_cycles,
                      levels=len(self.lv), status=status, rebuilds=rebuilds,
                      failed_mode=self.fail if self.fail is not None else -1)
        return f.A, report, np.array(trace)


DEFAULTS = dict(nu1_setup=5, nu2_setup=5, nuc_setup=100, n_test=2, nu1_solve=1, nu2_solve=1, nuc_solve=50,
                max_setup_cycles=5, min_setup_cycles=3, stagnation_eps=0.1, use_fmg=0, nu_fmg=50, fmg_guard=0,
                max_cycles=500, tol=1e-10, coarsest=0, solve_stagnation_after=5)


def mg_solve(Z, dims, A0, T0, A_fmg=None, **params):
    p = dict(DEFAULTS)
    p.update(params)
    R = A0[0].shape[1]
    return MGOracle(Z, dims, R, p).solve(A0, T0, A_fmg)


def als_solve(Z, dims, A0, tol=1e-10, max_iters=10000, check_every=1):
    """Standalone ALS: sweeps with normalization, g every check_every sweeps."""
    nz2 = float(np.vdot(Z, Z))
    A = [np.asfortranarray(a) for a in A0]
    g, it, status = float("nan"), 0, 1
    for it in range(1, max_iters + 1):
        A, _ = oracle.als_sweep(Z, dims, A, normZ2=nz2)
        A, _ = oracle.normalize_sort(dims, A, sort=False)
        if it % check_every == 0 or it == max_iters:
            g = oracle.gradient(Z, dims, A, normZ2=nz2, want_G=False)[0][1]
            if g < tol:
                status = 0
                break
    A, _ = oracle.normalize_sort(dims, A, sort=True)
    return A, dict(g=g, iterations=it, status=status)
