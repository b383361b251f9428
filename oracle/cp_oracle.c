/*
 * cp_oracle.c -- plain, slow, obviously-correct CPU fp64 ORACLE for the hot path of
 * De Sterck & Miller, "A multigrid method for low-rank canonical tensor decomposition"
 * (arXiv 1111.6091).  Citations "P:n" are line numbers of /root/reference/PAPER.md
 * (the paper's LaTeX source); equations are cited by their \label.
 *
 * ==> TEST INFRASTRUCTURE ONLY. <==
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  The product path (paper_1111_6091_b200/, libcp.so) never
 * calls, links or includes anything here, and this file includes nothing from it: the
 * two implementations share no code, headers, helpers or constants.
 *
 * Conventions (readings R2/R3):
 *   - a dense tensor Z of order N and size I_1 x ... x I_N is stored with mode 1
 *     fastest: linear index = sum_n i_n * prod_{k<n} I_k (0-based i_n);
 *   - a factor matrix A^(n) is I_n x R, column-major: A^(n)(i,r) = A[n][i + I_n*r];
 *   - every matrix argument (M, F, G, U, Gram) is column-major.
 * Arithmetic is IEEE binary64, no BLAS, no fast-math.  OpenMP is used only across
 * output rows / output entries whose own summation order is fixed, so results are
 * bitwise independent of the thread count.
 *
 * Status codes: 0 ok, -1 bad argument, -3 Cholesky pivot <= 0 (Gamma not SPD).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL (-1)
#define OR_ENOTSPD (-3)
#define OR_MAXN 8

/* element (i,r) of a column-major matrix with I rows */
#define CM(A, I, i, r) ((A)[(int64_t)(i) + (int64_t)(I) * (int64_t)(r)])

static int check_shape(int N, const int64_t *dims, int R) {
    if (N < 1 || N > OR_MAXN || R < 1 || !dims) return OR_EINVAL;
    for (int n = 0; n < N; ++n)
        if (dims[n] < 1) return OR_EINVAL;
    return OR_OK;
}

static int64_t numel(int N, const int64_t *dims) {
    int64_t p = 1;
    for (int n = 0; n < N; ++n) p *= dims[n];
    return p;
}

/* ||Z||^2, the squared Frobenius norm used in eq:CPfunctional. */
double oracle_norm2(int N, const int64_t *dims, const double *Z) {
    int64_t P = numel(N, dims);
    double s = 0.0;
    for (int64_t e = 0; e < P; ++e) s += Z[e] * Z[e];
    return s;
}

/*
 * MTTKRP  M = Z_(n) Phi^(n)   (eq:gradEqn P:104-107, eq:Phi P:109-111).
 * Z_(n) is the mode-n matricization: rows i_n, columns j enumerating the other
 * indices with the lowest remaining mode fastest, which matches the reversed Khatri-Rao
 * order of Phi^(n) = A^(N) (.) ... (.) A^(n+1) (.) A^(n-1) (.) ... (.) A^(1):
 * row j of Phi^(n) is Phi[j,r] = prod_{k != n} A^(k)(i_k, r).
 * Written out: M(i,r) = sum_j Z_(n)(i,j) * Phi(j,r), j ascending.
 * Fills rows [row_lo, row_hi) of M (I_n x R col-major); other rows untouched.
 */
int oracle_mttkrp_rows(int N, const int64_t *dims, int R, const double *Z,
                       const double *const *A, int mode, int64_t row_lo, int64_t row_hi,
                       double *M) {
    if (check_shape(N, dims, R) || mode < 0 || mode >= N || !Z || !A || !M) return OR_EINVAL;
    const int64_t In = dims[mode];
    if (row_lo < 0 || row_hi > In || row_lo > row_hi) return OR_EINVAL;
    for (int k = 0; k < N; ++k)
        if (k != mode && !A[k]) return OR_EINVAL;
    int64_t stride[OR_MAXN];
    stride[0] = 1;
    for (int k = 1; k < N; ++k) stride[k] = stride[k - 1] * dims[k - 1];
    const int64_t J = numel(N, dims) / In; /* number of columns of Z_(n) */

#pragma omp parallel
    {
        double *phi = (double *)malloc(sizeof(double) * (size_t)R);
        /* row i's R sums live in this thread-private array and are stored into M once: M is
         * column-major, so rows owned by different threads share cache lines (the summation
         * order -- j ascending per (i, r) -- is the same as accumulating in M) */
        double *acc = (double *)malloc(sizeof(double) * (size_t)R);
        int64_t idx[OR_MAXN];
#pragma omp for schedule(static)
        for (int64_t i = row_lo; i < row_hi; ++i) {
            for (int r = 0; r < R; ++r) acc[r] = 0.0;
            for (int k = 0; k < N; ++k) idx[k] = 0;
            for (int64_t j = 0; j < J; ++j) {
                /* idx holds the multi-index of column j (mode `mode` excluded) */
                int64_t lin = i * stride[mode];
                for (int k = 0; k < N; ++k)
                    if (k != mode) lin += idx[k] * stride[k];
                for (int r = 0; r < R; ++r) {
                    double p = 1.0;
                    for (int k = 0; k < N; ++k)
                        if (k != mode) p *= CM(A[k], dims[k], idx[k], r);
                    phi[r] = p;
                }
                const double z = Z[lin];
                for (int r = 0; r < R; ++r) acc[r] += z * phi[r];
                /* advance the column multi-index, lowest mode fastest */
                for (int k = 0; k < N; ++k) {
                    if (k == mode) continue;
                    if (++idx[k] < dims[k]) break;
                    idx[k] = 0;
                }
            }
            for (int r = 0; r < R; ++r) CM(M, In, i, r) = acc[r];
        }
        free(acc);
        free(phi);
    }
    return OR_OK;
}

int oracle_mttkrp(int N, const int64_t *dims, int R, const double *Z, const double *const *A,
                  int mode, double *M) {
    if (check_shape(N, dims, R) || mode < 0 || mode >= N) return OR_EINVAL;
    return oracle_mttkrp_rows(N, dims, R, Z, A, mode, 0, dims[mode], M);
}

/* Gram matrix Upsilon = A^T A, R x R. */
int oracle_gram(int64_t I, int R, const double *A, double *Ups) {
    if (I < 1 || R < 1 || !A || !Ups) return OR_EINVAL;
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < R; ++s) {
            double acc = 0.0;
            for (int64_t i = 0; i < I; ++i) acc += CM(A, I, i, r) * CM(A, I, i, s);
            CM(Ups, R, r, s) = acc;
        }
    return OR_OK;
}

/* Gamma^(n) = Upsilon^(1) * ... (skip n) ... * Upsilon^(N), Hadamard product (eq:Gamma P:113-116).
 * Ups is an array of N Gram matrices. */
int oracle_gamma(int N, int R, const double *const *Ups, int mode, double *Gam) {
    if (N < 1 || R < 1 || mode < 0 || mode >= N || !Ups || !Gam) return OR_EINVAL;
    for (int e = 0; e < R * R; ++e) {
        double p = 1.0;
        for (int k = 0; k < N; ++k)
            if (k != mode) p *= Ups[k][e];
        Gam[e] = p;
    }
    return OR_OK;
}

/* Textbook lower Cholesky Gamma = L L^T, no pivoting (reading R1: Cholesky replaces
 * the pseudoinverse of P:121; equal to it whenever Gamma is SPD).  L is R x R
 * column-major, upper triangle zeroed.  Returns OR_ENOTSPD on a pivot <= 0 (or NaN). */
int oracle_cholesky(int R, const double *G, double *L) {
    if (R < 1 || !G || !L) return OR_EINVAL;
    for (int e = 0; e < R * R; ++e) L[e] = 0.0;
    for (int j = 0; j < R; ++j) {
        double d = CM(G, R, j, j);
        for (int k = 0; k < j; ++k) d -= CM(L, R, j, k) * CM(L, R, j, k);
        if (!(d > 0.0)) return OR_ENOTSPD;
        const double ljj = sqrt(d);
        CM(L, R, j, j) = ljj;
        for (int i = j + 1; i < R; ++i) {
            double s = CM(G, R, i, j);
            for (int k = 0; k < j; ++k) s -= CM(L, R, i, k) * CM(L, R, j, k);
            CM(L, R, i, j) = s / ljj;
        }
    }
    return OR_OK;
}

/* Solve X Gamma = B row by row with Gamma = L L^T: for each row b (1 x R),
 * Gamma x^T = b^T (Gamma symmetric): forward L y = b^T, back L^T x^T = y.
 * B, X are I x R column-major (may alias). */
int oracle_solve_rows(int64_t I, int R, const double *L, const double *B, double *X) {
    if (I < 0 || R < 1 || !L || !B || !X) return OR_EINVAL;
    double *y = (double *)malloc(sizeof(double) * (size_t)R);
    for (int64_t i = 0; i < I; ++i) {
        for (int r = 0; r < R; ++r) {
            double s = CM(B, I, i, r);
            for (int k = 0; k < r; ++k) s -= CM(L, R, r, k) * y[k];
            y[r] = s / CM(L, R, r, r);
        }
        for (int r = R - 1; r >= 0; --r) {
            double s = y[r];
            for (int k = r + 1; k < R; ++k) s -= CM(L, R, k, r) * CM(X, I, i, k);
            CM(X, I, i, r) = s / CM(L, R, r, r);
        }
    }
    free(y);
    return OR_OK;
}

/*
 * One ALS / BNGS iteration (with a right-hand side F, eq:relaxinnersolve P:356-358):
 *   for n = 1..N (ascending, each step using the freshest factors, reading R4):
 *       M     = Z_(n) Phi^(n)                       (eq:gradEqn, eq:Phi)
 *       Gamma = *_{k != n} A^(k)^T A^(k)             (eq:Gamma)
 *       solve A^(n) Gamma = M + F^(n) by Cholesky    (P:121 with dagger -> Cholesky, reading R1)
 * No normalization or sorting here (reading R7: the driver does that, finest level only).
 * out[0] = f after the sweep by the expansion
 *          f = 1/2||Z||^2 - <M^(N), A^(N)> + 1/2 sum_{r,s} prod_k Upsilon^(k)_{rs}
 *   (M^(N) = Z_(N)Phi^(N) without F; <Z,[[A]]> = <Z_(N)Phi^(N), A^(N)> by eq:propMatricized
 *    and ||[[A]]||^2 = 1^T(*_k Upsilon^(k))1 by eq:Gamma; reading R6),
 * out[1] = f_tilde = f - sum_n <F^(n), A^(n)>   (the functional whose stationarity condition is
 *          H(A) = F, eq:FASfineprob; reading R5),
 * out[2] = status (0 or OR_ENOTSPD), out[3] = failed mode (0-based) or -1.
 * F may be NULL (all zero) or an array of N pointers, each NULL (= zero) or I_n x R.
 * normZ2 = ||Z||^2.  A is updated in place.
 */
int oracle_als_sweep(int N, const int64_t *dims, int R, const double *Z, double normZ2,
                     double *const *A, const double *const *F, double *out) {
    if (check_shape(N, dims, R) || !Z || !A || !out) return OR_EINVAL;
    for (int k = 0; k < N; ++k)
        if (!A[k]) return OR_EINVAL;
    out[0] = out[1] = NAN;
    out[2] = 0.0;
    out[3] = -1.0;
    double *Ups[OR_MAXN];
    for (int k = 0; k < N; ++k) {
        Ups[k] = (double *)malloc(sizeof(double) * (size_t)R * R);
        oracle_gram(dims[k], R, A[k], Ups[k]);
    }
    double *Gam = (double *)malloc(sizeof(double) * (size_t)R * R);
    double *L = (double *)malloc(sizeof(double) * (size_t)R * R);
    double *M = NULL, *Rhs = NULL;
    double inner_last = 0.0;
    int st = OR_OK;
    for (int n = 0; n < N; ++n) {
        const int64_t In = dims[n];
        M = (double *)malloc(sizeof(double) * (size_t)(In * R));
        Rhs = (double *)malloc(sizeof(double) * (size_t)(In * R));
        oracle_mttkrp(N, dims, R, Z, (const double *const *)A, n, M);
        for (int64_t e = 0; e < In * R; ++e)
            Rhs[e] = M[e] + ((F && F[n]) ? F[n][e] : 0.0);
        oracle_gamma(N, R, (const double *const *)Ups, n, Gam);
        st = oracle_cholesky(R, Gam, L);
        if (st != OR_OK) {
            out[2] = (double)st;
            out[3] = (double)n;
            free(M);
            free(Rhs);
            break;
        }
        oracle_solve_rows(In, R, L, Rhs, A[n]);
        oracle_gram(In, R, A[n], Ups[n]);
        if (n == N - 1) {
            inner_last = 0.0;
            for (int64_t e = 0; e < In * R; ++e) inner_last += M[e] * A[n][e];
        }
        free(M);
        free(Rhs);
    }
    if (st == OR_OK) {
        double model2 = 0.0; /* ||[[A]]||^2 = 1^T (*_k Ups^(k)) 1 */
        for (int e = 0; e < R * R; ++e) {
            double p = 1.0;
            for (int k = 0; k < N; ++k) p *= Ups[k][e];
            model2 += p;
        }
        const double f = 0.5 * normZ2 - inner_last + 0.5 * model2;
        double fa = 0.0;
        if (F)
            for (int n = 0; n < N; ++n)
                if (F[n])
                    for (int64_t e = 0; e < dims[n] * R; ++e) fa += F[n][e] * A[n][e];
        out[0] = f;
        out[1] = f - fa;
    }
    for (int k = 0; k < N; ++k) free(Ups[k]);
    free(Gam);
    free(L);
    return OR_OK; /* a numeric failure is reported through out[2], not the return code */
}

/* Model entry x = [[A]](i_1..i_N) = sum_r prod_n A^(n)(i_n, r)   (eq:tensorCP P:31-34). */
static double model_entry(int N, const int64_t *dims, int R, const double *const *A,
                          const int64_t *idx) {
    double x = 0.0;
    for (int r = 0; r < R; ++r) {
        double p = 1.0;
        for (int n = 0; n < N; ++n) p *= CM(A[n], dims[n], idx[n], r);
        x += p;
    }
    return x;
}

/* f = 1/2 ||Z - [[A]]||^2 by its definition (eq:CPfunctional P:38-42), element by element. */
double oracle_f_direct(int N, const int64_t *dims, int R, const double *Z, const double *const *A) {
    if (check_shape(N, dims, R) || !Z || !A) return NAN;
    const int64_t P = numel(N, dims);
    const int64_t I0 = dims[0];
    const int64_t cols = P / I0;
    double total = 0.0;
    /* per-column partial sums in fixed order, then summed in column order: thread-count
     * independent */
    double *colsum = (double *)malloc(sizeof(double) * (size_t)cols);
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < cols; ++q) {
        int64_t idx[OR_MAXN];
        int64_t t = q;
        for (int n = 1; n < N; ++n) {
            idx[n] = t % dims[n];
            t /= dims[n];
        }
        double s = 0.0;
        for (int64_t i = 0; i < I0; ++i) {
            idx[0] = i;
            const double d = Z[q * I0 + i] - model_entry(N, dims, R, A, idx);
            s += d * d;
        }
        colsum[q] = s;
    }
    for (int64_t q = 0; q < cols; ++q) total += colsum[q];
    free(colsum);
    return 0.5 * total;
}

/*
 * Gradient and stopping quantity at one iterate (eq:gradEqn P:104-107, eq:gradConv P:454-456):
 *   G^(n) = -Z_(n)Phi^(n) + A^(n) Gamma^(n)  [ - F^(n) when F is given: the FAS residual
 *           H^(n)(A) - F^(n), eq:FASop/eq:FASfineprob P:326-332 ]
 *   g = (sum_n ||G^(n)||^2)^{1/2} / ||Z||.
 * out[0] = f (direct, eq:CPfunctional), out[1] = g, out[2+n] = ||G^(n)||^2.
 * G: NULL or N pointers (each NULL or I_n x R) receiving G^(n).
 */
int oracle_gradient(int N, const int64_t *dims, int R, const double *Z, double normZ2,
                    const double *const *A, const double *const *F, double *out, double *const *G) {
    if (check_shape(N, dims, R) || !Z || !A || !out) return OR_EINVAL;
    double *Ups[OR_MAXN];
    for (int k = 0; k < N; ++k) {
        Ups[k] = (double *)malloc(sizeof(double) * (size_t)R * R);
        oracle_gram(dims[k], R, A[k], Ups[k]);
    }
    double *Gam = (double *)malloc(sizeof(double) * (size_t)R * R);
    double total = 0.0;
    for (int n = 0; n < N; ++n) {
        const int64_t In = dims[n];
        double *M = (double *)malloc(sizeof(double) * (size_t)(In * R));
        oracle_mttkrp(N, dims, R, Z, A, n, M);
        oracle_gamma(N, R, (const double *const *)Ups, n, Gam);
        double nrm = 0.0;
        for (int64_t i = 0; i < In; ++i)
            for (int r = 0; r < R; ++r) {
                double ag = 0.0;
                for (int s = 0; s < R; ++s) ag += CM(A[n], In, i, s) * CM(Gam, R, s, r);
                double gv = -CM(M, In, i, r) + ag;
                if (F && F[n]) gv -= CM(F[n], In, i, r);
                if (G && G[n]) CM(G[n], In, i, r) = gv;
                nrm += gv * gv;
            }
        out[2 + n] = nrm;
        total += nrm;
        free(M);
    }
    out[0] = oracle_f_direct(N, dims, R, Z, A);
    out[1] = sqrt(total) / sqrt(normZ2);
    for (int k = 0; k < N; ++k) free(Ups[k]);
    free(Gam);
    return OR_OK;
}

/*
 * n-mode product X = Z x_n U: U is J x I_n (column-major, U(j,i) = U[j + J*i]),
 * X has size I_1 x .. x J x .. x I_N and X_(n) = U Z_(n), i.e.
 *   X(i_1..j..i_N) = sum_{i=0}^{I_n-1} U(j,i) Z(i_1..i..i_N), i ascending.
 * The restriction of P:186-189 is U = Phat^T; interpolation (eq:CGC P:191) is the same call
 * on a 2-way factor matrix.
 */
int oracle_mode_product(int N, const int64_t *dims, const double *Z, int mode, const double *U,
                        int64_t J, double *X) {
    if (N < 1 || N > OR_MAXN || !dims || mode < 0 || mode >= N || J < 1 || !Z || !U || !X)
        return OR_EINVAL;
    for (int n = 0; n < N; ++n)
        if (dims[n] < 1) return OR_EINVAL;
    int64_t left = 1, right = 1;
    for (int k = 0; k < mode; ++k) left *= dims[k];
    for (int k = mode + 1; k < N; ++k) right *= dims[k];
    const int64_t In = dims[mode];
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < right; ++b)
        for (int64_t j = 0; j < J; ++j)
            for (int64_t a = 0; a < left; ++a) {
                double s = 0.0;
                for (int64_t i = 0; i < In; ++i)
                    s += CM(U, J, j, i) * Z[a + left * (i + In * b)];
                X[a + left * (j + J * b)] = s;
            }
    return OR_OK;
}

/*
 * Normalization eq:ALSnorm: lambda_r = (prod_n ||a_r^(n)||)^{1/N},
 * a_r^(n) <- lambda_r a_r^(n) / ||a_r^(n)||; then the rank-one terms are sorted in
 * decreasing order of lambda_r, stable (ties keep index order).
 * lambda (R) receives the sorted lambdas.  A zero column leaves the factors unchanged
 * for that component (lambda_r = 0).
 */
int oracle_normalize(int N, const int64_t *dims, int R, double *const *A, double *lambda, int sort) {
    if (check_shape(N, dims, R) || !A || !lambda) return OR_EINVAL;
    double *lam = (double *)malloc(sizeof(double) * (size_t)R);
    for (int r = 0; r < R; ++r) {
        double nrm[OR_MAXN];
        double prod = 1.0;
        for (int n = 0; n < N; ++n) {
            double s = 0.0;
            for (int64_t i = 0; i < dims[n]; ++i) s += CM(A[n], dims[n], i, r) * CM(A[n], dims[n], i, r);
            nrm[n] = sqrt(s);
            prod *= nrm[n];
        }
        lam[r] = pow(prod, 1.0 / (double)N);
        if (prod > 0.0)
            for (int n = 0; n < N; ++n)
                for (int64_t i = 0; i < dims[n]; ++i)
                    CM(A[n], dims[n], i, r) = lam[r] * (CM(A[n], dims[n], i, r) / nrm[n]);
    }
    /* stable insertion sort of the component order by decreasing lambda */
    int *ord = (int *)malloc(sizeof(int) * (size_t)R);
    for (int r = 0; r < R; ++r) ord[r] = r;
    for (int a = 1; sort && a < R; ++a) {
        int v = ord[a];
        int b = a - 1;
        while (b >= 0 && lam[ord[b]] < lam[v]) {
            ord[b + 1] = ord[b];
            --b;
        }
        ord[b + 1] = v;
    }
    for (int n = 0; n < N; ++n) {
        const int64_t In = dims[n];
        double *tmp = (double *)malloc(sizeof(double) * (size_t)(In * R));
        for (int r = 0; r < R; ++r)
            for (int64_t i = 0; i < In; ++i) CM(tmp, In, i, r) = CM(A[n], In, i, ord[r]);
        memcpy(A[n], tmp, sizeof(double) * (size_t)(In * R));
        free(tmp);
    }
    for (int r = 0; r < R; ++r) lambda[r] = lam[ord[r]];
    free(ord);
    free(lam);
    return OR_OK;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int oracle_normalize_sort(int N, const int64_t *dims, int R, double *const *A, double *lambda) {
    return oracle_normalize(N, dims, R, A, lambda, 1);
}

/* set the OpenMP thread count (tests check that results are bitwise thread-count independent) */
void oracle_set_threads(int n) {
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    omp_set_num_threads(n);
#else
    (void)n;
#endif
}
