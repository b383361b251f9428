// small_kernels.cu -- the R x R side of the hot path (eq:Gamma P:113-116, Cholesky solve of
// P:121 / eq:relaxinnersolve P:356-358, the functional eq:CPfunctional P:38-42, the gradient
// eq:gradEqn and g eq:gradConv P:454-456) plus ||Z||^2.  All reductions run in a fixed order
// (no atomics), so results are bitwise reproducible.  These kernels are latency-bound: every
// global read is issued in independent batches, and the R x R algebra runs in registers of
// one warp (R is a template parameter).
#include "small_kernels.cuh"
#ifdef CP_SOLVE_TIMING
#include <cstdio>
#endif

namespace cpk {

// sum of n strided values, 8 independent loads in flight, combined in a fixed order
__device__ __forceinline__ double sum_strided(const double *p, int64_t stride, int n) {
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int c = 0;
  for (; c + 8 <= n; c += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] += p[(int64_t)(c + j) * stride];
  }
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (c + j < n) s[j] += p[(int64_t)(c + j) * stride];
  return ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
}

// ---------------------------------------------------------------- reduction of stream partials
// Part j of sp of the fixed-order sum that forms M(i, r) from the stream kernel's partials.
__device__ __forceinline__ double reduce_entry_part(const ReduceGeom &g, int64_t i, int r, int j, int sp) {
  if (g.direct) return (j == 0) ? g.part[i + g.In_rows * r] : 0.0;
  if (g.mode0) {  // mode 0: one I1 x R partial per column group; chunk j of the groups
    const int c0 = (int)(((int64_t)g.Gc * j) / sp), c1 = (int)(((int64_t)g.Gc * (j + 1)) / sp);
    return sum_strided(g.part + (int64_t)c0 * g.I1 * g.R + i + g.I1 * r, g.I1 * g.R, c1 - c0);
  }
  if (j != 0) return 0.0;
  // mode m >= 1: R-vector partials per (column group, row block, segment)
  double s = 0.0;
  const int64_t lo = i * g.Qn, hi = (i + 1) * g.Qn - 1;
  const int64_t clo = ((lo + 1) * g.Gc - 1) / g.Q;
  const int64_t chi = ((hi + 1) * g.Gc - 1) / g.Q;
  for (int64_t c = clo; c <= chi; ++c) {
    const int64_t seg_first = ((c * g.Q) / g.Gc) / g.Qn;
    for (int rb = 0; rb < g.RB; ++rb) s += g.part[(((c * g.RB + rb) * g.slots) + (i - seg_first)) * g.R + r];
  }
  return s;
}

// Phase A of the solve / gradient kernels: M rows [i0, i0 + nrows) into sM (row-major, R per
// row), using sp threads per entry.  Needs a 256-double scratch.
__device__ void gather_rows(const ReduceGeom &g, int64_t i0, int nrows, int R, int sp, double *sM,
                            double *scratch) {
  const int tid = threadIdx.x;
  const int ent = tid / sp, j = tid - (tid / sp) * sp;
  double v = 0.0;
  if (ent < nrows * R) {
    const int ii = ent / R, r = ent - (ent / R) * R;
    v = reduce_entry_part(g, i0 + ii, r, j, sp);
  }
  if (sp == 1) {
    if (ent < nrows * R) sM[ent] = v;
    return;
  }
  scratch[tid] = v;
  __syncthreads();
  if (j == 0 && ent < nrows * R) {
    double s = 0.0;
    for (int k = 0; k < sp; ++k) s += scratch[tid + k];
    sM[ent] = s;
  }
}

__global__ void __launch_bounds__(256) reduce_mttkrp_kernel(const ReduceGeom g, int rpc, int sp, double *M) {
  griddep();
  __shared__ double sM[256], scratch[256];
  const int64_t i0 = (int64_t)blockIdx.x * rpc;
  const int nrows = (int)((g.In_rows - i0) < rpc ? (g.In_rows - i0) : rpc);
  gather_rows(g, i0, nrows, g.R, sp, sM, scratch);
  __syncthreads();
  for (int e = threadIdx.x; e < nrows * g.R; e += blockDim.x) {
    const int ii = e / g.R, r = e - (e / g.R) * g.R;
    M[(i0 + ii) + g.In_rows * r] = sM[e];
  }
}

// cp_mttkrp, mode 0: M[e] = sum_c part[c * S + e] over the Gc column-group partials, e = i + I*r
// (the partial and the output share the column-major layout).  A 1024-thread block covers 32
// consecutive e (coalesced 256-byte rows) x 32 fixed chunks of c (~Gc/32 loads per thread, all
// in flight: one or two memory round trips), combined in chunk order.
__global__ void __launch_bounds__(1024) reduce_mode0_kernel(const double *part, int Gc, int64_t S, double *M) {
  griddep();
  __shared__ double red[32][33];
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lx;
  const int c0 = (Gc * ly) / 32, c1 = (Gc * (ly + 1)) / 32;
  red[ly][lx] = (e < S) ? sum_strided(part + (int64_t)c0 * S + e, S, c1 - c0) : 0.0;
  __syncthreads();
  if (ly == 0 && e < S) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k) t += red[k][lx];
    M[e] = t;
  }
}

// ---------------------------------------------------------------- prep: At copies + Grams
// One block per (mode k, chunk of kPrepRows rows): At^(k) rows (row-major copy, padded stride
// RS) and the chunk's partial Gram A_chunk^T A_chunk, summed later in chunk order.
__global__ void __launch_bounds__(256) prep_kernel(const PrepArgs a) {
  CTL_BEGIN
  griddep();
  CTL_AFTER_WAIT
  // chunk x R, column-major (r * kPrepLd + ii); the odd column stride keeps the Gram loop's
  // 16 different r of a warp in 16 different banks (stride 64 put them all in one bank)
  constexpr int kPrepLd = kPrepRows + 1;
  __shared__ double sA[kPrepLd * 32];
  int k = 0;
  while (k + 1 < a.N && (int)blockIdx.x >= a.blk_off[k + 1]) ++k;
  const int b = blockIdx.x - a.blk_off[k];
  const int R = a.R, RS = R + (R & 1), RR = R * R;
  const int64_t I = a.dims[k];
  const double *A = a.A[k];
  const int tid = threadIdx.x;
  if (blockIdx.x == 0 && tid == 0 && a.status != nullptr) {
    if (!a.keep_status) {
      a.status[0] = 0.0;
      a.status[1] = -1.0;
    }
    *reinterpret_cast<unsigned *>(a.status + kTicketSlot) = 0u;  // solve completion ticket
    *reinterpret_cast<unsigned *>(a.status + kTicketSlot2) = 0u;  // ylsolve ticket
  }
  if (blockIdx.x == 0 && a.zero != nullptr)
    for (int i = tid; i < a.nzero; i += blockDim.x) a.zero[i] = 0u;
  if (A == nullptr) return;
  double *At = a.At[k];
  const int64_t i0 = (int64_t)b * kPrepRows;
  const int n = (int)((I - i0) < kPrepRows ? (I - i0) : kPrepRows);
  for (int e = tid; e < n * R; e += blockDim.x) {
    const int r = e / n, ii = e - (e / n) * n;
    sA[r * kPrepLd + ii] = A[(i0 + ii) + I * r];
  }
  __syncthreads();
  for (int e = tid; e < n * RS; e += blockDim.x) {
    const int ii = e / RS, r = e - (e / RS) * RS;
    At[(i0 + ii) * RS + r] = (r < R) ? sA[r * kPrepLd + ii] : 0.0;
  }
  if (a.gpre != nullptr) {
    for (int e = tid; e < RR; e += blockDim.x) {
      const int r = e % R, s = e / R;
      const double *ar = sA + r * kPrepLd, *as = sA + s * kPrepLd;
      // 4 independent chains (the single 64-long fma chain dominated this kernel)
      double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
      int ii = 0;
      for (; ii + 3 < n; ii += 4) {
        g0 = fma(ar[ii], as[ii], g0);
        g1 = fma(ar[ii + 1], as[ii + 1], g1);
        g2 = fma(ar[ii + 2], as[ii + 2], g2);
        g3 = fma(ar[ii + 3], as[ii + 3], g3);
      }
      for (; ii < n; ++ii) g0 = fma(ar[ii], as[ii], g0);
      a.gpre[(int64_t)blockIdx.x * RR + e] = (g0 + g1) + (g2 + g3);
    }
  }
  CTL_END("prep")
}

// Upsilon^(k) entry e from the prep partials of mode k (fixed chunk order)
__device__ __forceinline__ double prep_gram(const PrepGrams &pg, int k, int e, int RR) {
  if (pg.tot != nullptr) return pg.tot[(int64_t)k * RR + e];
  return sum_strided(pg.gpre + (int64_t)pg.blk_off[k] * RR + e, RR, pg.nblk[k]);
}

// ---------------------------------------------------------------- sweep finalize: f, f_tilde
// f = 1/2 ||Z||^2 - <M^(N), A^(N)> + 1/2 1^T (*_k Upsilon^(k)) 1 (reading R6) and
// f~ = f - sum_n <F^(n), A^(n)> (reading R5); run by one 256-thread block.
__device__ void finalize_body(const FinalizeArgs &a, double *sred) {
  const int R = a.R, RR = R * R, tid = threadIdx.x;
  if (a.status[0] != 0.0) {
    if (tid == 0) {
      a.out[0] = nan("");
      a.out[1] = nan("");
      a.out[2] = a.status[0];
      a.out[3] = a.status[1];
    }
    return;
  }
  // Upsilon^(N) from the last solve's partials; ||[[A]]||^2 = 1^T (*_k Upsilon^(k)) 1.  All
  // loads are issued before the one combined block reduction.
  double m2 = 0.0;
  for (int e = tid; e < RR; e += blockDim.x) {
    double p = 1.0;
    for (int k = 0; k < a.N - 1; ++k) p *= a.Ups[(int64_t)k * RR + e];
    const double u = sum_strided(a.glast + e, RR, a.nlast);
    a.Ups[(int64_t)(a.N - 1) * RR + e] = u;
    m2 = fma(u, p, m2);
  }
  double in = 0.0;
  for (int c = tid; c < a.nlast; c += blockDim.x) in += a.dotM_last[c];
  double fl = 0.0;
  for (int n = 0; n < a.N; ++n)
    for (int c = tid; c < a.nsolve[n]; c += blockDim.x) fl += a.dotF[(int64_t)n * a.dot_stride + c];
  block_sum3_256(m2, in, fl, sred);
  const double model2 = m2, inner = in, fa = fl;
  if (tid == 0) {
    const double f = 0.5 * a.normZ2[0] - inner + 0.5 * model2;
    a.out[0] = f;
    a.out[1] = f - fa;
    a.out[2] = 0.0;
    a.out[3] = -1.0;
  }
}

__global__ void __launch_bounds__(256) finalize_sweep_kernel(const FinalizeArgs a) {
  griddep();
  __shared__ double sred[256];
  finalize_body(a, sred);
}

// ---------------------------------------------------------------- per-mode solve (sweep)
// One warp factors Gamma = L L^T in registers (lane i holds row i) and forms L^{-1}; every
// row of A^(n) is then x = L^{-T} (L^{-1} (m + f)) as two small triangular mat-vecs.  With
// a.fin_on (the sweep's last solve) the last block to finish also runs finalize_body
// (completion ticket; every sum keeps its fixed order, so results stay bitwise reproducible).
#ifdef CP_SOLVE_TIMING
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SOLVE_T(k) if (threadIdx.x == 0) tstamp[k] = gtimer();
#else
#define SOLVE_T(k)
#endif
template <int R>
__global__ void __launch_bounds__(256) solve_kernel_t(const SolveArgs a) {
#ifdef CP_SOLVE_TIMING
  unsigned long long tstamp[10] = {0};
#endif
  SOLVE_T(0);
  CTL_BEGIN
  griddep();
  CTL_AFTER_WAIT
  SOLVE_T(1);
  constexpr int RR = R * R;
  constexpr int LS = R + 1;  // smem row stride of the R x R matrices
  __shared__ double sL[R * LS];    // Gamma, then L (lower)
  __shared__ double sLi[R * LS];   // L^{-1} (lower)
  __shared__ double sDi[R];        // 1 / L(j, j)
  __shared__ double sUp[RR];
  __shared__ double sM[256], sB[256], sX[256], scratch[256];
  __shared__ int sfail;
  __shared__ unsigned sticket;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool live = (a.status[0] == 0.0);  // an earlier mode already failed: straight to the ticket
  if (live) {
    const int64_t In = a.In;
    const int64_t i0 = (int64_t)blockIdx.x * a.rpc;
    const int nrows = (int)((In - i0) < a.rpc ? (In - i0) : a.rpc);
    if (a.linv != nullptr) {
      // L^{-1} from the Gamma job (gamma_job.cuh); the Gram totals are in Ups already
      for (int e = tid; e < RR; e += blockDim.x) sLi[(e / R) * LS + (e % R)] = a.linv[e];
    } else if (a.gprev != nullptr && !(a.dbg & 1)) {
      // total Gram of the previous mode from its per-CTA partials (fixed order)
      for (int e = tid; e < RR; e += blockDim.x) {
        const double s = sum_strided(a.gprev + e, RR, a.nprev);
        sUp[e] = s;
        if (blockIdx.x == 0) a.Ups[(int64_t)a.prev_mode * RR + e] = s;
      }
    }
    SOLVE_T(2);
    // phase A (independent of Gamma): M rows from the stream partials
    gather_rows(a.rg, i0, nrows, R, a.sp, sM, scratch);
    __syncthreads();
    SOLVE_T(3);
    if (a.linv == nullptr) {
      // Gamma^(n) = *_{k != n} Upsilon^(k)   (eq:Gamma).  Upsilon^(k): k > n from the prep
      // partials (factor not yet updated in this sweep), k = n-1 from the previous solve's
      // partials, k < n-1 from the totals the earlier solves wrote.
      for (int e = tid; e < RR; e += blockDim.x) {
        double gm = 1.0;
        if (a.dbg & 1) {
          sL[(e % R) * LS + (e / R)] = ((e % R) == (e / R)) ? 1.0 : 0.0;
          continue;
        }
        for (int k = 0; k < a.N; ++k) {
          if (k == a.mode) continue;
          double u;
          if (k > a.mode) u = prep_gram(a.pg, k, e, RR);
          else if (k == a.prev_mode) u = sUp[e];
          else u = a.Ups[(int64_t)k * RR + e];
          gm *= u;
        }
        sL[(e % R) * LS + (e / R)] = gm;
      }
    }
    for (int e = tid; e < nrows * R; e += blockDim.x) {
      const int ii = e / R, r = e - (e / R) * R;
      sB[e] = sM[e] + (a.F != nullptr ? a.F[(i0 + ii) + In * r] : 0.0);
    }
    if (tid == 0) sfail = 0;
    __syncthreads();
    SOLVE_T(4);
    if (a.linv != nullptr) {
      // (factored by the Gamma job)
    } else if (warp == 0 && (a.dbg & 1)) {
      for (int k = 0; k < R; ++k)
        if (lane < R) sLi[lane * LS + k] = (k == lane) ? 1.0 : 0.0;
    } else if (warp == 0) {
      // Cholesky, right-looking, lane i = row i (no pivoting; fail on a pivot <= 0 or NaN).
      // 1/L(j,j) = rsqrt(pivot) and L(j,j) = pivot * rsqrt(pivot): no divisions on the chain.
      double g[R];
#pragma unroll
      for (int k = 0; k < R; ++k) g[k] = (lane < R) ? sL[lane * LS + k] : 0.0;
      bool ok = true;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const double piv = __shfl_sync(0xffffffffu, g[j], j);
        if (!(piv > 0.0)) {
          ok = false;
          break;
        }
        const double inv = rsqrt(piv);
        if (lane == 0) sDi[j] = inv;
        if (lane == j) g[j] = piv * inv;
        else if (lane > j) g[j] *= inv;
#pragma unroll
        for (int k = j + 1; k < R; ++k) {
          const double lkj = __shfl_sync(0xffffffffu, g[j], k);
          if (lane >= k) g[k] = fma(-g[j], lkj, g[k]);
        }
      }
      if (!ok) {
        if (lane == 0) sfail = 1;
      } else {
#pragma unroll
        for (int k = 0; k < R; ++k)
          if (lane < R) sL[lane * LS + k] = (k <= lane) ? g[k] : 0.0;
        __syncwarp();
        // L^{-1}: lane c forms column c by forward substitution
        double x[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
          double s = (i == lane) ? 1.0 : 0.0;
#pragma unroll
          for (int k = 0; k < i; ++k) s = fma(-sL[i * LS + k], x[k], s);
          x[i] = (i >= lane) ? s * sDi[i] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < R; ++i)
          if (lane < R) sLi[i * LS + lane] = x[i];
      }
    }
    __syncthreads();
    SOLVE_T(5);
    if (sfail) {
      if (blockIdx.x == 0 && tid == 0) {
        a.status[0] = (double)CP_ENOTSPD;
        a.status[1] = (double)a.mode;
      }
    } else {
      // y = L^{-1} b, then x = L^{-T} y, thread per (row, r)
      for (int e = tid; e < nrows * R; e += blockDim.x) {
        const int ii = e / R, r = e - (e / R) * R;
        double y = 0.0;
#pragma unroll 4
        for (int k = 0; k <= r; ++k) y = fma(sLi[r * LS + k], sB[ii * R + k], y);
        scratch[e] = y;
      }
      __syncthreads();
      double dm = 0.0, df = 0.0;
      for (int e = tid; e < nrows * R; e += blockDim.x) {
        const int ii = e / R, r = e - (e / R) * R;
        double x = 0.0;
#pragma unroll 4
        for (int k = r; k < R; ++k) x = fma(sLi[k * LS + r], scratch[ii * R + k], x);
        const int64_t i = i0 + ii;
        a.A[i + In * r] = x;
        a.At[i * (R + (R & 1)) + r] = x;
        sX[e] = x;
        dm = fma(sM[e], x, dm);
        if (a.F != nullptr) df = fma(a.F[i + In * r], x, df);
      }
      SOLVE_T(6);
      // partial Gram of the new rows, and the CTA's <M,A>, <F,A> (fixed order)
      double dms = dm, dfs = df, unused = 0.0;
      block_sum3_256(dms, dfs, unused, scratch);
      SOLVE_T(7);
      for (int e = tid; e < RR; e += blockDim.x) {
        const int r = e % R, s = e / R;
        double g0 = 0.0, g1 = 0.0;
        int ii = 0;
        for (; ii + 1 < nrows; ii += 2) {
          g0 = fma(sX[ii * R + r], sX[ii * R + s], g0);
          g1 = fma(sX[(ii + 1) * R + r], sX[(ii + 1) * R + s], g1);
        }
        if (ii < nrows) g0 = fma(sX[ii * R + r], sX[ii * R + s], g0);
        a.gcur[(int64_t)blockIdx.x * RR + e] = g0 + g1;
      }
      if (tid == 0) {
        a.dotM[blockIdx.x] = dms;
        a.dotF[blockIdx.x] = dfs;
      }
    }
  }
  if (a.fin_on) {
    __threadfence();
    __syncthreads();
    if (tid == 0) sticket = atomicAdd(a.ticket, 1u);
    __syncthreads();
    if (sticket == gridDim.x - 1) {
      __threadfence();
      finalize_body(a.fin, scratch);
      if (tid == 0) *a.ticket = 0u;
    }
  }
  SOLVE_T(8);
  CTL_END("solve")
#ifdef CP_SOLVE_TIMING
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
    printf("solve mode %d blk %d: griddep %llu | pre %llu gather %llu gamma %llu chol %llu apply %llu gram/dot %llu tail %llu\n",
           a.mode, blockIdx.x, tstamp[1] - tstamp[0], tstamp[2] - tstamp[1], tstamp[3] - tstamp[2], tstamp[4] - tstamp[3],
           tstamp[5] - tstamp[4], tstamp[6] - tstamp[5], tstamp[7] - tstamp[6], tstamp[8] - tstamp[7]);
#endif
}

// ---------------------------------------------------------------- gradient (cp_fit)
// G^(n)(i,r) = -M(i,r) + sum_s A(i,s) Gamma(s,r) - F(i,r)   (eq:gradEqn; FAS residual with F)
__global__ void __launch_bounds__(256) gradient_kernel(const GradArgs a) {
  griddep();
  __shared__ double sG[32 * 32];
  __shared__ double sM[256], scratch[256];
  const int R = a.R, RR = R * R, tid = threadIdx.x;
  for (int e = tid; e < RR; e += blockDim.x) {
    double gm = 1.0;
    for (int k = 0; k < a.N; ++k)
      if (k != a.mode) gm *= prep_gram(a.pg, k, e, RR);
    sG[e] = gm;
  }
  const int64_t In = a.In;
  const int64_t i0 = (int64_t)blockIdx.x * a.rpc;
  const int nrows = (int)((In - i0) < a.rpc ? (In - i0) : a.rpc);
  gather_rows(a.rg, i0, nrows, R, a.sp, sM, scratch);
  __syncthreads();
  double g2 = 0.0, dm = 0.0;
  for (int e = tid; e < nrows * R; e += blockDim.x) {
    const int ii = e / R, r = e - (e / R) * R;
    const int64_t i = i0 + ii;
    double gv = -sM[e];
    for (int s = 0; s < R; ++s) gv = fma(a.A[i + In * s], sG[s + R * r], gv);
    if (a.F != nullptr) gv -= a.F[i + In * r];
    if (a.G != nullptr) a.G[i + In * r] = gv;
    g2 = fma(gv, gv, g2);
    if (a.dpart != nullptr) dm = fma(sM[e], a.A[i + In * r], dm);
  }
  const double t = block_sum_256(g2, scratch);
  if (tid == 0) a.gpart[blockIdx.x] = t;
  if (a.dpart != nullptr) {
    const double d = block_sum_256(dm, scratch);
    if (tid == 0) a.dpart[blockIdx.x] = d;
  }
}

__global__ void __launch_bounds__(256) finalize_fit_kernel(const FitFinalArgs a) {
  griddep();
  __shared__ double sred[256];
  const int tid = threadIdx.x;
  double rs = 0.0;
  for (int c = tid; c < a.nresid; c += blockDim.x) rs += a.resid[c];
  const double res = block_sum_256(rs, sred);
  double tot = 0.0;
  for (int n = 0; n < a.N; ++n) {
    double s = 0.0;
    for (int c = tid; c < a.ngrad[n]; c += blockDim.x) s += a.gpart[(int64_t)n * a.gstride + c];
    const double sn = block_sum_256(s, sred);
    if (tid == 0) a.out[2 + n] = sn;
    tot += sn;
  }
  double f = 0.5 * res;
  if (a.expand) {
    // f = 1/2 ||Z||^2 - <M^(N), A^(N)> + 1/2 ||[[A]]||^2 (reading R6), fixed summation order
    const int RR = a.R * a.R;
    double m2 = 0.0, in = 0.0, unused = 0.0;
    for (int e = tid; e < RR; e += blockDim.x) {
      double p = 1.0;
      for (int k = 0; k < a.N; ++k) p *= prep_gram(a.pg, k, e, RR);
      m2 += p;
    }
    for (int c = tid; c < a.ndot; c += blockDim.x) in += a.dpart[c];
    block_sum3_256(m2, in, unused, sred);
    f = 0.5 * a.normZ2[0] - in + 0.5 * m2;
  }
  if (tid == 0) {
    a.out[0] = f;
    a.out[1] = sqrt(tot) / sqrt(a.normZ2[0]);
  }
}

// ---------------------------------------------------------------- ||Z||^2
__global__ void __launch_bounds__(512) norm2_kernel(const double *__restrict__ Z, int64_t P,
                                                    double *part) {
  griddep();
  __shared__ double sred[512];
  const int tid = threadIdx.x;
  double s0 = 0.0, s1 = 0.0;
  const int64_t n2 = P / 2;
  const double2 *Z2 = reinterpret_cast<const double2 *>(Z);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + tid; e < n2; e += stride) {
    const double2 z = __ldg(Z2 + e);
    s0 = fma(z.x, z.x, s0);
    s1 = fma(z.y, z.y, s1);
  }
  if (blockIdx.x == 0 && tid == 0 && (P & 1)) s0 = fma(Z[P - 1], Z[P - 1], s0);
  sred[tid] = s0 + s1;
  __syncthreads();
  for (int off = 256; off > 0; off >>= 1) {
    if (tid < off) sred[tid] += sred[tid + off];
    __syncthreads();
  }
  if (tid == 0) part[blockIdx.x] = sred[0];
}

__global__ void __launch_bounds__(256) norm2_final_kernel(const double *part, int n, double *out) {
  griddep();
  __shared__ double sred[256];
  double s = 0.0;
  for (int c = threadIdx.x; c < n; c += blockDim.x) s += part[c];
  const double t = block_sum_256(s, sred);
  if (threadIdx.x == 0) out[0] = t;
}

// ---------------------------------------------------------------- dimension-tree sweep helpers
// After the Y_L pass, every segment i1 that a CTA boundary splits has its contributions in the
// edge blocks of the CTAs c_lo..c_hi that cover it; block (c, chunk) completes the segment
// holding v0(c) (the first boundary inside that segment does the work), summing the edge blocks
// in CTA order into yl.  Afterwards yl holds Y_L(:, i1, :) for every i1.  The contributing
// edge blocks are located once per block (shared table); the element loop is plain 32-bit math.
__global__ void __launch_bounds__(256) yl_fixup_kernel(const YLGeom y, int chunks) {
  griddep();
  constexpr int kMaxContrib = 64;
  __shared__ int64_t soff[kMaxContrib];
  const int64_t c = blockIdx.x / chunks + 1;
  const int chunk = blockIdx.x % chunks;
  const int64_t v0c = (c * y.Q) / y.Gc;
  const int64_t s = v0c / y.Qn;
  if (v0c % y.Qn == 0) return;                      // boundary on a segment edge: nothing split
  const int64_t v0p = ((c - 1) * y.Q) / y.Gc;
  if (v0p > s * y.Qn) return;                       // an earlier boundary in s handles it
  const int64_t clo = ((s * y.Qn + 1) * y.Gc - 1) / y.Q;
  const int64_t chi = (((s + 1) * y.Qn) * y.Gc - 1) / y.Q;
  const int nc = (int)(chi - clo + 1);
  const int64_t blk = y.I0 * y.R;
  for (int k = threadIdx.x; k < nc && k < kMaxContrib; k += blockDim.x) {
    const int64_t cc = clo + k;
    const int64_t seg_first = ((cc * y.Q) / y.Gc) / y.Qn;
    soff[k] = (cc * y.RB * 2 + ((seg_first == s) ? 0 : 1)) * blk;
  }
  __syncthreads();
  const int I0 = (int)y.I0;
  const int e0 = (int)((blk * chunk) / chunks), e1 = (int)((blk * (chunk + 1)) / chunks);
  for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const int rb = (y.RB == 1) ? 0 : (e % I0) / y.Wmax;
    const double *src = y.edge + (int64_t)rb * 2 * blk + e;
    double acc = 0.0;
    int k = 0;
    for (; k < nc && k < kMaxContrib; ++k) acc += src[soff[k]];
    for (; k < nc; ++k) {  // (more than kMaxContrib CTAs share one segment: tiny tensors only)
      const int64_t cc = clo + k;
      const int64_t seg_first = ((cc * y.Q) / y.Gc) / y.Qn;
      acc += src[(cc * y.RB * 2 + ((seg_first == s) ? 0 : 1)) * blk];
    }
    ((double *)y.yl)[s * blk + e] = acc;
  }
}

// Partials of M0(i0, r) = sum_{i1} Y_L(i0, i1, r) A^(1)(i1, r).  Block (b, r) sums the i1 of
// range b (of S ranges); warp w takes the i1 = w (mod 8) of the range and reads whole 4-KB
// Y_L(:, i1, r) rows (lane -> i0 = lane + 32 k, 16 k per chunk of 512 rows); the 8 warp sums
// combine in warp order into part[b][r][i0] -- the layout of the mode-0 MTTKRP partials, summed
// in range order by the mode-0 solve (ReduceGeom mode0, Gc = S).
__global__ void __launch_bounds__(256) ymm0_kernel(const YLGeom y, const double *A1, int S, double *part) {
  griddep();
  __shared__ double sred[8][512];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b = blockIdx.x, r = blockIdx.y;
  const int64_t blk = y.I0 * y.R;
  const int64_t a0 = (y.I1 * b) / S, a1 = (y.I1 * (b + 1)) / S;
  const double *ap = A1 + y.I1 * r;
  for (int64_t c0 = 0; c0 < y.I0; c0 += 512) {
    double acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = 0.0;
    const double *yr0 = y.yl + y.I0 * r + c0 + lane;
    const int nk = (int)((y.I0 - c0 + 31 - lane) / 32);  // rows of this lane in the chunk
    for (int64_t i1 = a0 + w; i1 < a1; i1 += 8) {
      const double av = ap[i1];
      const double *yp = yr0 + i1 * blk;
      if (nk >= 16) {
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] = fma(yp[32 * k], av, acc[k]);
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (k < nk) acc[k] = fma(yp[32 * k], av, acc[k]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) sred[w][lane + 32 * k] = acc[k];
    __syncthreads();
    for (int e = threadIdx.x; e < 512 && c0 + e < y.I0; e += blockDim.x) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) t += sred[k][e];
      part[((int64_t)b * y.R + r) * y.I0 + c0 + e] = t;
    }
  }
}

// M1(i1, r) = sum_{i0} Y_L(i0, i1, r) A^(0)(i0, r): warp per (r, 4 consecutive i1), lanes stride
// over i0 (contiguous in Y_L and in the column-major A0; each A0 value feeds 4 rows), 4
// independent partial sums per row, fixed shuffle tree
__global__ void __launch_bounds__(256) ymm1_kernel(const YLGeom y, const double *A0, double *M1,
                                                   const GammaJob gj) {
  griddep();
  if (gj.on && blockIdx.x == gridDim.x - 1) {  // extra block: Gamma^(1) for the next solve
    __shared__ double gsm[gamma_job_smem_doubles(32)];
    gamma_job_run(gj, gsm, threadIdx.x, blockDim.x, true);
    return;
  }
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nq = (y.I1 + 3) / 4;
  if (wg >= nq * y.R) return;
  const int r = (int)(wg / nq);
  const int64_t i1b = (wg - (int64_t)r * nq) * 4;
  const int64_t blk = y.I0 * y.R;
  const double *ap = A0 + y.I0 * r;
  const double *yp = y.yl + i1b * blk + y.I0 * r;
  int nu = (int)(y.I1 - i1b);
  if (nu > 4) nu = 4;
  double s[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int j = 0; j < 4; ++j) s[u][j] = 0.0;
  for (int64_t i0 = lane; i0 < y.I0; i0 += 128) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t idx = i0 + 32 * j;
      if (idx < y.I0) {
        const double a = ap[idx];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (u < nu) s[u][j] = fma(yp[u * blk + idx], a, s[u][j]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    double t = (s[u][0] + s[u][1]) + (s[u][2] + s[u][3]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if (lane == 0 && u < nu) M1[i1b + u + y.I1 * r] = t;
  }
}

// warp per (i_m, r): lanes stride over the other indices j of modes 2..N-1
__global__ void __launch_bounds__(256) yr_kernel(const YRArgs a) {
  griddep();
  if (a.gj.on && blockIdx.x == gridDim.x - 1) {  // extra block: Gamma^(mode) for the next solve
    __shared__ double gsm[gamma_job_smem_doubles(32)];
    gamma_job_run(a.gj, gsm, threadIdx.x, blockDim.x, true);
    return;
  }
  const int64_t Im = a.dims[a.mode];
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= Im * a.R) return;
  const int64_t im = w % Im;
  const int r = (int)(w / Im);
  int64_t J = 1;
  for (int k = 2; k < a.N; ++k) J *= a.dims[k];
  const int64_t nother = J / Im;
  double s = 0.0;
  for (int64_t o = lane; o < nother; o += 32) {
    // o enumerates the indices of modes 2..N-1 except mode, lowest mode fastest
    int64_t t = o, j = 0, stride = 1;
    double wgt = 1.0;
    for (int k = 2; k < a.N; ++k) {
      int64_t ik;
      if (k == a.mode) {
        ik = im;
      } else {
        ik = t % a.dims[k];
        t /= a.dims[k];
        wgt *= a.At[k][ik * a.RS + r];
      }
      j += ik * stride;
      stride *= a.dims[k];
    }
    s = fma(a.YR[j + J * r], wgt, s);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) a.M[im + Im * r] = s;
}

cudaError_t launch_yl_fixup(const YLGeom &y, cudaStream_t st) {
  if (y.Gc < 2) return cudaSuccess;
  int chunks = (int)((y.I0 * y.R + 2047) / 2048);
  if (chunks > 16) chunks = 16;
  return launch_k(yl_fixup_kernel, dim3((unsigned)((y.Gc - 1) * chunks)), dim3(256), 0, st, y, chunks);
}

int ymm0_ranges(int R, int64_t I1) {
  int S = (296 + R - 1) / R;  // about two blocks per SM
  if (S > 32) S = 32;
  if (S > I1) S = (int)I1;
  return S < 1 ? 1 : S;
}

void ymm0_solve_blocking(int R, int64_t I1, int *rpc, int *sp) {
  // one thread per M0 entry (sums the <= 32 range partials, 8 loads in flight): keeps the solve
  // grid -- and so the number of Gram partials the next solve sums -- small
  (void)I1;
  const int r = 256 / R;
  *sp = 1;
  *rpc = r < 1 ? 1 : r;
}

cudaError_t launch_ymm0(const YLGeom &y, const double *A1, double *part, cudaStream_t st) {
  const int S = ymm0_ranges(y.R, y.I1);
  return launch_k(ymm0_kernel, dim3((unsigned)S, (unsigned)y.R), dim3(256), 0, st, y, A1, S, part);
}

cudaError_t launch_ymm1(const YLGeom &y, const double *A0, double *M1, const GammaJob &gj, cudaStream_t st) {
  const int64_t threads = ((y.I1 + 3) / 4) * y.R * 32;
  const unsigned grid = (unsigned)((threads + 255) / 256) + (gj.on ? 1u : 0u);
  return launch_k(ymm1_kernel, dim3(grid), dim3(256), 0, st, y, A0, M1, gj);
}

cudaError_t launch_yr(const YRArgs &a, cudaStream_t st) {
  const int64_t threads = a.dims[a.mode] * a.R * 32;
  return launch_k(yr_kernel, dim3((unsigned)((threads + 255) / 256) + (a.gj.on ? 1u : 0u)), dim3(256), 0, st, a);
}

// ---------------------------------------------------------------- host-side launchers
template <int R>
static cudaError_t launch_solve_t(const SolveArgs &a, int grid, cudaStream_t st) {
  return launch_k(solve_kernel_t<R>, dim3(grid), dim3(256), 0, st, a);
}

cudaError_t launch_solve(const SolveArgs &a, int grid, cudaStream_t st) {
  switch (a.R) {
#define CPK_SOLVE_CASE(r) \
  case r: return launch_solve_t<r>(a, grid, st);
    CPK_SOLVE_CASE(1) CPK_SOLVE_CASE(2) CPK_SOLVE_CASE(3) CPK_SOLVE_CASE(4) CPK_SOLVE_CASE(5)
    CPK_SOLVE_CASE(6) CPK_SOLVE_CASE(7) CPK_SOLVE_CASE(8) CPK_SOLVE_CASE(9) CPK_SOLVE_CASE(10)
    CPK_SOLVE_CASE(11) CPK_SOLVE_CASE(12) CPK_SOLVE_CASE(13) CPK_SOLVE_CASE(14) CPK_SOLVE_CASE(15)
    CPK_SOLVE_CASE(16) CPK_SOLVE_CASE(17) CPK_SOLVE_CASE(18) CPK_SOLVE_CASE(19) CPK_SOLVE_CASE(20)
    CPK_SOLVE_CASE(21) CPK_SOLVE_CASE(22) CPK_SOLVE_CASE(23) CPK_SOLVE_CASE(24) CPK_SOLVE_CASE(25)
    CPK_SOLVE_CASE(26) CPK_SOLVE_CASE(27) CPK_SOLVE_CASE(28) CPK_SOLVE_CASE(29) CPK_SOLVE_CASE(30)
    CPK_SOLVE_CASE(31) CPK_SOLVE_CASE(32)
#undef CPK_SOLVE_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_prep(const PrepArgs &a, cudaStream_t st) {
  return launch_k(prep_kernel, dim3(a.blk_off[a.N]), dim3(256), 0, st, a);
}

}  // namespace cpk
