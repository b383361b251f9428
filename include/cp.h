/*
 * cp.h -- C ABI of libcp.so, the B200 (sm_100a) hot path of the multigrid CP method of
 * De Sterck & Miller, arXiv 1111.6091 ("P:n" = line n of the paper's LaTeX source).
 *
 * The library computes, on one GPU, in IEEE fp64:
 *   cp_mttkrp        M = Z_(n) Phi^(n)                       eq:gradEqn, eq:Phi
 *   cp_als_sweep(s)  one (or nsweeps) ALS / BNGS iteration(s) (with optional   P:121, eq:relaxinnersolve P:356-358
 *                    FAS right-hand side F) and the functional f  eq:CPfunctional P:38-42
 *   cp_mode_product  X = Z x_n U (restriction U = Phat^T,      P:74-78, eq:ctensor_transformed
 *                    interpolation on a 2-way factor matrix)
 *   cp_restrict_structured  X = Z x_n Phat^T for the BAMG
 *                    transfer operator (bidiagonal factor, O(P))
 *   cp_fit           f (direct), g and ||G^(n)||^2              eq:gradConv P:454-456
 *   cp_gradient      g, ||G^(n)||^2, G^(n) and f (expansion)    eq:gradEqn, eq:gradConv; SURVEY NEXT-2
 *                    at one iterate, without the residual pass
 *   cp_norm2         ||Z||^2
 *
 * ---------------------------------------------------------------------------------------
 * Conventions
 *   - Every pointer is DEVICE memory unless marked [host].  The caller owns every buffer,
 *     the workspace included; the library allocates nothing and frees nothing.
 *   - Tensor layout: Z of size I_1 x ... x I_N is dense, mode 1 fastest:
 *       linear index = sum_n i_n * prod_{k<n} I_k        (0-based i_n; Kolda-Bader order,
 *     consistent with the reversed Khatri-Rao order of Phi^(n)).
 *   - Matrix layout: A^(n), M, F, G (I_n x R) and U (J x I_n) are column-major:
 *       entry (i, r) at i + rows * r.
 *   - Modes are 0-based in this ABI (mode 0 = the paper's mode 1).
 *   - Limits: 1 <= N <= CP_MAX_N (cp_mode_product; N >= 2 for the others),
 *     1 <= R <= CP_MAX_R, every I_n >= 1, prod I_n < 2^62.
 *   - Inputs are never modified, except A in cp_als_sweep.  Outputs must not alias inputs.
 *   - Nothing synchronizes the host: all work is enqueued on `stream` (a cudaStream_t;
 *     NULL = legacy default stream), so whole sweeps can be captured in a CUDA graph.
 *     A workspace may be used by one stream at a time.
 *   - Results are deterministic: no atomics in any reduction, fixed summation order, so two
 *     runs on the same inputs are bitwise identical.
 *
 * Errors
 *   - Argument / shape errors return synchronously, before anything is enqueued:
 *       CP_EINVAL  null pointer, N or R out of range, mode out of range, J < 1
 *       CP_EDIM    a dimension < 1 or the element count overflows
 *       CP_EWORKSPACE  ws_bytes smaller than the matching *_workspace_bytes()
 *   - CP_ECUDA: a launch failed (cudaGetLastError after enqueueing).
 *   - Numeric failures are asynchronous: a non-positive Cholesky pivot (Gamma singular, e.g.
 *     a zero factor column -- the Keller condition of P:362) is written into the device
 *     `out` status word as CP_ENOTSPD together with the failing mode; the factors are then
 *     unspecified.
 *
 * Environment
 *   The shipped library reads a fixed list of PATH SELECTORS from the environment on each call
 *   (path_flag() in csrc/capi.cu; everything else -- tuning and debugging knobs -- exists only in
 *   -DCP_EXPERIMENTS builds).  A selector switches between implementations of the same operation
 *   whose results agree bitwise or within the parity tolerance; each one is exercised by the GPU
 *   parity tests.  Unset = the default in brackets:
 *     CP_STREAM_MMA [1]      0: DFMA register-tile consumers instead of the FP64 tensor-core ones
 *     CP_RESID_MMA [1]       0: DFMA residual pass in cp_fit
 *     CP_STREAM_TMAP [1]     0: one bulk copy per Z column instead of one tensor-map TMA per stage
 *     CP_STREAM_LEAN [1]     0: full-feature streaming kernels also for plans that need no feature
 *     CP_STREAM_PREFETCH [1 up to 2^26 elements]  Z of the first stages issued before the PDL wait
 *     CP_SWEEP_TREE [1]      0: one Z pass per mode instead of the two-pass dimension tree
 *     CP_SWEEP_TAIL [1 up to 2^26 elements]  last mode solved inside the mode-2 pass (2: every sweep)
 *     CP_YLSOLVE [1]         0: separate contraction and solve kernels for modes 0 and 1
 *     CP_SMALL_SWEEP [1], CP_TINY_SWEEP [1], CP_SWEEPS_GRAD_FUSED [1]  fused kernels of small tensors
 *     CP_MTTKRP_FCM [1], CP_MTTKRP_FUSED [1]  cp_mttkrp: factor rows from the caller's factors, one launch
 *     CP_MODEPROD_DMMA [1], CP_MODEPROD_PIPE [1]  mode products: tensor-core GEMM, cp.async ring
 *     CP_MG_GRAPH [1], CP_ALS_GRAPH [1], CP_MG_STRUCTURED [1]  host driver: CUDA graphs, structured restriction
 *     CP_PDL [1]             0: no programmatic dependent launch
 */
#ifndef CP_H
#define CP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CP_MAX_N 8
#define CP_MAX_R 32
#define CP_VERSION 1

enum {
    CP_OK = 0,
    CP_EINVAL = -1,
    CP_EDIM = -2,
    CP_ENOTSPD = -3,
    CP_ECUDA = -4,
    CP_EWORKSPACE = -5
};

/* a cudaStream_t (struct CUstream_st*), spelled without including the CUDA headers */
typedef struct CUstream_st *cp_stream_t;

/* [host] problem shape: order N, rank R, sizes dims[0..N-1] (= I_1..I_N) */
typedef struct {
    int32_t N;
    int32_t R;
    int64_t dims[CP_MAX_N];
} cp_shape;

/* Workspace bytes needed by cp_norm2 / cp_mttkrp / cp_als_sweep / cp_fit for shape s on the
 * current device (depends on the SM count).  0 on an invalid shape. */
size_t cp_workspace_bytes(const cp_shape *s);

/* ||Z||^2 -> out[0] (device).  The squared Frobenius norm of eq:CPfunctional. */
int cp_norm2(const cp_shape *s, const double *Z, double *out, void *ws, size_t ws_bytes,
             cp_stream_t stream);

/* MTTKRP  M = Z_(mode) Phi^(mode)   (eq:gradEqn P:104-107, eq:Phi P:109-111)
 *   A    [host] array of N device pointers to I_k x R factors (A[mode] is not read and may be
 *        NULL);  M: I_mode x R, column-major, overwritten.
 *   M(i,r) = sum over all other indices of z * prod_{k != mode} A^(k)(i_k, r).  The Khatri-
 *   Rao product Phi is never materialized; Z is streamed from HBM exactly once. */
int cp_mttkrp(const cp_shape *s, const double *Z, const double *const *A, int32_t mode,
              double *M, void *ws, size_t ws_bytes, cp_stream_t stream);

/* One ALS / block nonlinear Gauss-Seidel sweep -- with a right-hand side, the BNGS
 * relaxation of the FAS solve phase (eq:relaxinnersolve P:356-358):
 *   for n = 0..N-1 (ascending; each update uses the freshest factors):
 *       M = Z_(n) Phi^(n);  Gamma = *_{k != n} A^(k)^T A^(k)   (eq:Gamma P:113-116)
 *       A^(n) <- (M + F^(n)) Gamma^{-1}   via Gamma = L L^T, L lower, no pivoting.
 *   Z       tensor (the finest tensor or a coarse-level tensor, eq:cfunc P:181-185)
 *   normZ2  device pointer to ||Z||^2 (from cp_norm2)
 *   A       [host] N device pointers, I_n x R each, updated in place
 *   F       [host] NULL (all zero) or N device pointers, each NULL (= 0) or I_n x R
 *   out     device, 4 doubles: f, f_tilde, status (CP_OK or CP_ENOTSPD), failed mode or -1
 *           f       = 1/2 ||Z - [[A]]||^2 after the sweep, evaluated without another pass as
 *                     1/2||Z||^2 - <M^(N),A^(N)> + 1/2 sum_{r,s} prod_k (A^(k)^T A^(k))_{rs}
 *           f_tilde = f - sum_n <F^(n), A^(n)>  (the functional minimized block-wise when F != 0)
 *   No normalization or sorting (the driver does that on the finest level only). */
int cp_als_sweep(const cp_shape *s, const double *Z, const double *normZ2, double *const *A,
                 const double *const *F, double *out, void *ws, size_t ws_bytes,
                 cp_stream_t stream);

/* nsweeps >= 1 consecutive cp_als_sweep calls (the nu relaxations of a multigrid level, Table 1
 * P:462-478), out = the values after the last sweep (f, f~ before any normalization); a numeric
 * failure stops at the failing sweep.  flags: 0, or CP_SWEEPS_NORMALIZE = each sweep followed
 * by the eq:ALSnorm normalization without sorting (= cp_normalize_sort(sort = 0)), the
 * ALS relaxation of the setup phase.  For a tensor small enough to live in one CTA's shared
 * memory (P <= 16384, the coarse levels) all nsweeps (and normalizations) run in ONE launch of a
 * fused kernel; otherwise it loops the general sweep (+ cp_normalize_sort).  Same arguments and
 * errors as cp_als_sweep (nsweeps < 1 or unknown flags: CP_EINVAL). */
#define CP_SWEEPS_NORMALIZE 1
int cp_als_sweeps(const cp_shape *s, const double *Z, const double *normZ2, double *const *A,
                  const double *const *F, int32_t nsweeps, int32_t flags, double *out, void *ws,
                  size_t ws_bytes, cp_stream_t stream);

/* n-mode product X = Z x_mode U  (X_(n) = U Z_(n))
 *   dims [host] N sizes of Z;  U: J x dims[mode], column-major;  X: dims with dims[mode] -> J.
 *   Restriction (coarse tensor, Alg. 1 step 7 P:273): U = Phat^T;  interpolation A = Phat A_c
 *   (eq:CGC P:191): N = 2, dims = {I_c, R}, mode 0, U = Phat.
 *   ws may be NULL when cp_mode_product_workspace_bytes() returns 0. */
size_t cp_mode_product_workspace_bytes(int32_t N, const int64_t *dims, int32_t mode, int64_t J);
int cp_mode_product(int32_t N, const int64_t *dims, const double *Z, int32_t mode,
                    const double *U, int64_t J, double *X, void *ws, size_t ws_bytes,
                    cp_stream_t stream);

/* Restriction by the structured transfer operator of the geometric C/F splitting (SURVEY
 * 8(f) NEXT-3):  X = Z x_mode Phat^T,  Phat = P L^{-T},  B = P^T P = L L^T   (P:164-189,
 * eq:ctensor_transformed P:176-180; Phat^T Phat = I).
 *   P (I x Ic, I = dims[mode], Ic = ceil(I/2)) is the interpolation of P:222-247: the C points
 *   are the even 0-based fine indices (the paper's odd points), P(2j, j) = 1 (injection); the
 *   F point i = 2j+1 interpolates from its coarse neighbours,
 *       P(i, j) = wl[i],   P(i, j+1) = wr[i]   (wr is ignored when i = I-1: one-sided right end)
 *   -- the weights of Algorithm 1's weighted least-squares fit (eq:LSQinterp).  Entries of wl,
 *   wr at C points are ignored.
 *   Because P has at most two nonzeros per row, B is tridiagonal and L bidiagonal: the library
 *   factors B on the device and applies Phat^T = L^{-1} P^T along mode `mode` as a 3-point
 *   gather and a bidiagonal forward substitution per fiber -- O(P) flops and one pass over Z
 *   (HBM-bound), instead of the 2 * Ic * P flops of cp_mode_product with a dense Phat^T.  The
 *   result equals cp_mode_product(N, dims, Z, mode, Phat^T, Ic, ...) up to rounding.
 *   wl, wr  device, I doubles each
 *   X       device, the tensor with dims[mode] replaced by Ic (same layout as Z)
 *   ws      device workspace of cp_restrict_workspace_bytes() bytes (the factor of B)
 *   Errors: CP_EINVAL (null pointer, N out of [1, CP_MAX_N], mode out of range), CP_EDIM,
 *   CP_EWORKSPACE, CP_ECUDA.  B is SPD for any finite weights (every coarse point has its
 *   injected C row), so there is no numeric failure mode. */
size_t cp_restrict_workspace_bytes(int32_t N, const int64_t *dims, int32_t mode);
int cp_restrict_structured(int32_t N, const int64_t *dims, const double *Z, int32_t mode,
                           const double *wl, const double *wr, double *X, void *ws, size_t ws_bytes,
                           cp_stream_t stream);

/* Fit and stopping quantity at one iterate (eq:gradConv P:454-456):
 *   out  device, 2 + N doubles: f (direct, one residual pass over Z), g, ||G^(n)||^2 (n < N)
 *        G^(n) = -Z_(n)Phi^(n) + A^(n)Gamma^(n) [- F^(n)]  (eq:gradEqn; with F the FAS residual
 *        H^(n)(A) - F^(n), eq:FASop P:326-328);  g = (sum_n ||G^(n)||^2)^{1/2} / ||Z||
 *   F    [host] NULL or N device pointers (entries may be NULL)
 *   G    [host] NULL or N device pointers (entries may be NULL) receiving G^(n), I_n x R. */
int cp_fit(const cp_shape *s, const double *Z, const double *normZ2, const double *const *A,
           const double *const *F, double *out, double *const *G, void *ws, size_t ws_bytes,
           cp_stream_t stream);

/* All-modes gradient at one iterate (eq:gradEqn, eq:gradConv P:454-456): every
 * M^(n) = Z_(n)Phi^(n) with the SAME factors (no Gauss-Seidel dependency), so for N >= 3 the
 * dimension tree reads Z twice for all N modes (a Y_L pass and a mode-2 pass), and no residual
 * pass.  This is what the multigrid driver needs for the stopping test g and the FAS operator
 * H(A) (eq:FASop P:326-328, eq:FASrhs P:398).  Same arguments and G as cp_fit; out differs only
 * in out[0]:
 *   out  device, 2 + N doubles: f by the expansion f = 1/2 ||Z||^2 - <M^(N), A^(N)>
 *        + 1/2 1^T (*_k A^(k)T A^(k)) 1 (reading R6; equals cp_fit's direct f up to cancellation
 *        of order eps * ||Z||^2), g, ||G^(n)||^2 (n < N).  F enters G only, as in cp_fit.
 *   Errors: as cp_fit. */
int cp_gradient(const cp_shape *s, const double *Z, const double *normZ2, const double *const *A,
                const double *const *F, double *out, double *const *G, void *ws, size_t ws_bytes,
                cp_stream_t stream);

/* cp_als_sweeps followed by cp_gradient(F = gF) at the new iterate -- the pair every level of a
 * CP-FAS V-cycle issues (Algorithm 2: relax, then H(A) for eq:FASrhs).  The results
 * (A, out, gout, G) are bitwise those of the two separate calls; on tensors that run the fused
 * shared-memory sweep kernel the gradient pass runs in the same launch (Z and the factors are
 * loaded once).
 *   out   as cp_als_sweeps (4 doubles);  gout, G, gF as out, G, F of cp_gradient (gout: 2 + N
 *   doubles; if the sweeps fail with CP_ENOTSPD in out, gout[0..1] are NaN)
 *   Errors: as cp_als_sweeps. */
int cp_als_sweeps_then_gradient(const cp_shape *s, const double *Z, const double *normZ2,
                                double *const *A, const double *const *F, int32_t nsweeps,
                                int32_t flags, double *out, const double *const *gF, double *gout,
                                double *const *G, void *ws, size_t ws_bytes, cp_stream_t stream);

/* Number of kernel launches the last successful call on this thread enqueued (for the
 * benchmark's gpu_launches count). */
int cp_last_launch_count(void);

/* Live per-kernel timing for the roofline report.  While enabled, every launch of the
 * Z-streaming kernel (the MTTKRP / residual pass that dominates the sweep) is bracketed by a
 * pair of CUDA events recorded on the launch stream (at most 8192 pairs are kept).
 * cp_profile_read synchronizes on the recorded events and returns, for the launches recorded
 * since the last read: their count, the summed event durations in ms, and the summed
 * ALGORITHMIC bytes (8P + 8R*sum_{k != n} I_k + 8 I_n R per MTTKRP launch);
 * then it resets.  Host-side only; not thread-safe. */
int cp_profile_enable(int enable);
int cp_profile_read(int64_t *launches, double *total_ms, double *alg_bytes);

/* ---------------------------------------------------------------------------------------
 * Normalization and ordering of the factors (eq:ALSnorm P:122-125; sort P:126):
 *   lambda_r = (prod_n ||a_r^(n)||)^{1/N},  a_r^(n) <- lambda_r a_r^(n) / ||a_r^(n)||;
 *   a component with a zero column is left unchanged (lambda_r = 0);
 *   if sort != 0 the components are reordered by decreasing lambda (stable).
 *   A [host] N device pointers (in/out);  lambda: device, R doubles, or NULL.
 *   Workspace: cp_workspace_bytes(s) suffices. */
int cp_normalize_sort(const cp_shape *s, double *const *A, int32_t sort, double *lambda, void *ws,
                      size_t ws_bytes, cp_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * Multigrid driver (host C++ on top of the calls above):
 * the BAMG setup V-cycle CP-AMG-mult (Algorithm 1) with geometric coarsening
 * and weighted least-squares interpolation (eq:LSQinterp, eq:interpweights
 * P:236-247), the Cholesky-transformed Galerkin coarse tensors (eq:ctensor_transformed), the
 * CP-FAS solve V-cycle (Algorithm 2), FMG-CP-FAS (Algorithm 3) and the
 * setup/solve combination with the stagnation rules of P:486-492.  Every level's work runs in
 * the kernels of this library; the host builds P, B = P^T P, its Cholesky factor and
 * Phat = P L^{-T} (O(I * I_c)) and reads g once per cycle.  This call synchronizes the stream. */
typedef struct {
    int32_t nu1_setup, nu2_setup, nuc_setup, n_test; /* Table 1: 5, 5, 100, 2 */
    int32_t nu1_solve, nu2_solve, nuc_solve;          /* 1, 1, 50 */
    int32_t max_setup_cycles, min_setup_cycles;       /* 5, 3 */
    double stagnation_eps;                            /* 0.1 (eq:stagnation) */
    int32_t use_fmg, nu_fmg;                          /* "Multilevel + FMG"; coarsest ALS its */
    int32_t max_cycles;                               /* 500 multilevel iterations */
    double tol;                                       /* tau (1e-10) */
    int32_t coarsest;                                 /* I_coarsest; 0 = 2R (reading R16) */
    int32_t solve_stagnation_after;                   /* 5 */
    int32_t max_trace;                                /* rows of the trace buffer */
    int32_t fmg_guard;                                /* 0 (default): P:492 -- the solve phase always
                                                         continues from the FMG result, after a
                                                         down-sweep rebuild of the operators;
                                                         1: reading R29 -- keep the FMG result only
                                                         if it lowers g (else restore the setup
                                                         iterate, no rebuild) */
} cp_mg_params;

void cp_mg_default_params(cp_mg_params *p);
size_t cp_mg_workspace_bytes(const cp_shape *s, const cp_mg_params *p);
/* Z: finest tensor;  A: [host] N device pointers, boot factor matrices (initial guess in,
 * solution out);  T: [host] n_test*N device pointers, initial test factor matrices (block t,
 * mode n at T[t*N + n]; read only);  A_fmg: [host] N device pointers to the coarsest-level
 * random initial guess of FMG (ignored unless use_fmg);  report [host, 16 doubles]:
 *   0 g, 1 f, 2 cycles (setup + FMG + solve), 3 setup cycles, 4 solve cycles, 5 levels,
 *   6 status (0 converged, 1 cycle limit, CP_ENOTSPD: a relaxation on some level hit a
 *   non-positive Cholesky pivot -- the solve stops at the next stopping test), 7 trace rows,
 *   8 rebuilds, 9 seconds, 10 device seconds of the stopping tests (excluded from the paper's
 *   timings), 11 failing mode of a CP_ENOTSPD (else -1);
 * trace [host, max_trace x 4]: phase (0 setup, 1 FMG, 2 solve), cycle, g, seconds.
 * Reentrant: all driver state is per call (the workspace and the heap). */
int cp_mg_solve(const cp_shape *s, const double *Z, double *const *A, const double *const *T,
                const double *const *A_fmg, const cp_mg_params *prm, double *report, double *trace,
                void *ws, size_t ws_bytes, cp_stream_t stream);

/* Standalone ALS (the paper's baseline): sweeps with normalization until g < tol or
 * max_iters; g is evaluated every `check_every` sweeps, together with the status word of every
 * sweep since the last check.  report [host, 8]: 0 g, 1 f, 2 iterations, 3 status (0 converged,
 * 1 iteration limit, CP_ENOTSPD: a sweep hit a non-positive Cholesky pivot -- the loop stops at
 * the next check), 4 seconds, 5 seconds of the stopping tests, 6 failing mode (or -1). */
size_t cp_als_solve_workspace_bytes(const cp_shape *s);
int cp_als_solve(const cp_shape *s, const double *Z, double *const *A, double tol, int32_t max_iters,
                 int32_t check_every, double *report, void *ws, size_t ws_bytes, cp_stream_t stream);

const char *cp_status_string(int code);
int cp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CP_H */
