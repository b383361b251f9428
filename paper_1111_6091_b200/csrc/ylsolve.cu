// ylsolve.cu -- modes 0 and 1 of the dimension-tree sweep in one kernel each: the contraction of
// Y_L with one factor (M^(0) or M^(1), eq:gradEqn P:104-111 via the dimension tree, DESIGN 6.5),
// Gamma^(n) = *_{k != n} Upsilon^(k) (eq:Gamma P:113-116), its Cholesky factor (reading R1) and
// the row solves A^(n) Gamma^(n) = M^(n) + F^(n) (eq:relaxinnersolve P:356-358).
//
// Y_L(i0, i1, r) = sum_{i_2..} z * prod_{k>=2} A^(k)(i_k, r) is stored [i1][r][i0] (yl).
//   mode 0:  M0(i0, r) = sum_{i1} Y_L(i0, i1, r) A^(1)(i1, r)      (A^(1) of the previous sweep)
//   mode 1:  M1(i1, r) = sum_{i0} Y_L(i0, i1, r) A^(0)_new(i0, r)  (Gauss-Seidel order, R4)
// A block owns kRows output rows and forms them completely (no partial outputs, no second
// kernel): the mode-0 block reads the 32-byte pieces Y_L(i0b..i0b+3, i1, r) for every (i1, r),
// the mode-1 block the contiguous rows Y_L(:, i1, r) of its i1.  Gamma is summed from Gram
// partials and factored by warp 0 in registers while nothing depends on it (every block
// repeats this R x R work -- it is cheaper than a grid-wide dependency).  The new rows' partial
// Grams (and <F, A>) are reduced across each 8-CTA cluster through distributed shared memory
// in CTA-rank order, so the next consumer sums one partial per cluster.  All sums run in a
// fixed order: results are bitwise reproducible.
#include <cooperative_groups.h>

#include "small_kernels.cuh"
#ifdef CP_SOLVE_TIMING
#include <cstdio>
#define YS_T(k) \
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tst[k]));
#else
#define YS_T(k)
#endif

namespace cg = cooperative_groups;

namespace cpk {

constexpr int kYsRows = 4;     // output rows per block
constexpr int kYsCluster = 8;  // CTAs per cluster (partial-Gram reduction)

// sum of n strided values, 8 independent loads in flight, combined in a fixed order
__device__ __forceinline__ double ys_sum(const double *p, int64_t stride, int n) {
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

// 32-byte load (LDG.256 on sm_100a); p must be 32-B aligned
__device__ __forceinline__ void ld_v4(const double *p, double (&v)[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}
// kYsRows consecutive doubles (the block's rows of one Y_L column) in one vector load
template <int N>
__device__ __forceinline__ void ld_rows(const double *p, double (&v)[N]) {
  if constexpr (N == 4) {
    ld_v4(p, v);
  } else {
    static_assert(N == 2, "kYsRows: 2 or 4");
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "l"(p));
  }
}

// Gamma^(mode)(e) for the entries e = lane + 32 q of one warp: products of Upsilon^(k), k !=
// mode, read as totals (Ups, bit k of a.ups_total; all loads of a lane issued before use) or
// summed in a fixed order from partials (mode 1, k = 0: the cluster partials gin; else the prep
// partials of the old factor; block 0 writes those sums to Ups).
constexpr int kYsMaxF = CP_MAX_N - 1;
template <int R>
__device__ __forceinline__ void ys_gamma_warp(const YLSolveArgs &a, double *sL, const double *sU0, int lane) {
  constexpr int RR = R * R, LS = R + 1, NQ = (RR + 31) / 32;
  if (a.ups_total == (((1 << a.N) - 1) & ~(1 << a.mode))) {
    double v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[q] = 1.0;
    for (int k = 0; k < a.N; ++k) {
      if (k == a.mode) continue;
      const double *src = (a.mode == 1 && k == 0 && a.nin > 0) ? sU0 : a.Ups + (int64_t)k * RR;
      double t[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) t[q] = (lane + 32 * q < RR) ? src[lane + 32 * q] : 1.0;
#pragma unroll
      for (int q = 0; q < NQ; ++q) v[q] *= t[q];
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int e = lane + 32 * q;
      if (e < RR) sL[(e % R) * LS + (e / R)] = v[q];
    }
    return;
  }
  for (int e = lane; e < RR; e += 32) {
    double gm = 1.0;
    for (int k = 0; k < a.N; ++k) {
      if (k == a.mode) continue;
      double u;
      if (a.ups_total & (1 << k)) {
        u = a.Ups[(int64_t)k * RR + e];
      } else {
        u = (a.mode == 1 && k == 0) ? ys_sum(a.gin + e, RR, a.nin)
            : (a.pg.tot != nullptr ? a.pg.tot[(int64_t)k * RR + e]
                                   : ys_sum(a.pg.gpre + (int64_t)a.pg.blk_off[k] * RR + e, RR, a.pg.nblk[k]));
        if (blockIdx.x == 0) a.Ups[(int64_t)k * RR + e] = u;
      }
      gm *= u;
    }
    sL[(e % R) * LS + (e / R)] = gm;
  }
}

// 1/sqrt(x) for x > 0: the MUFU approximation (rsqrt.approx.f64) and two Newton steps in
// fp64 -- inline, no slow-path call (CUDA's rsqrt(double) calls a subroutine whose register
// save/restore dominated the factorization inside the solve kernels).
__device__ __forceinline__ double ys_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx, y * y, 1.5);
  y = y * fma(-hx, y * y, 1.5);
  return y;
}

// Cholesky Gamma = L L^T by one warp (lane i = row i; no pivoting; a non-positive or NaN pivot
// sets *fail) and L^{-1} by forward substitution (lane c = column c); 1/L(j,j) = ys_rsqrt(pivot).
template <int R>
__device__ __forceinline__ void ys_chol_warp(double *sL, double *sLi, double *sDi, int *fail, int lane) {
  constexpr int LS = R + 1;
  double g[R];
#pragma unroll
  for (int k = 0; k < R; ++k) g[k] = (lane < R) ? sL[lane * LS + k] : 0.0;
  bool ok = true;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const double piv = __shfl_sync(0xffffffffu, g[j], j);
    ok = ok && (piv > 0.0);
    const double inv = ys_rsqrt(ok ? piv : 1.0);
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
    if (lane == 0) *fail = 1;
    return;
  }
#pragma unroll
  for (int k = 0; k < R; ++k)
    if (lane < R) sL[lane * LS + k] = (k <= lane) ? g[k] : 0.0;
  __syncwarp();
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

template <int R>
__global__ void __launch_bounds__(256, 2) __cluster_dims__(kYsCluster, 1, 1) ylsolve_kernel_t(const YLSolveArgs a) {
#ifdef CP_SOLVE_TIMING
  unsigned long long tst[10] = {0};
#endif
  YS_T(0);
  CTL_BEGIN
  griddep();
  CTL_AFTER_WAIT
  constexpr int RR = R * R;
  constexpr int LS = R + 1;
  constexpr int NSL = 256 / R;        // mode 0: i1 slices (8 contraction warps)
  constexpr int EPW = (kYsRows * R + 6) / 7;  // mode 1: entries per contraction warp (7 or 8 warps)
  __shared__ double sL[R * LS];    // Gamma, then L (lower)
  __shared__ double sLi[R * LS];   // L^{-1}
  __shared__ double sDi[R];
  __shared__ double sB[kYsRows * R], sY[kYsRows * R], sX[kYsRows * R], sMv[kYsRows * R];
  __shared__ double sP[NSL * R * kYsRows];  // mode 0: per-slice row sums
  __shared__ double sGram[RR];
  __shared__ double sDot[8];
  __shared__ int sfail;
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t In = a.In;
  const int64_t r0 = (int64_t)blockIdx.x * kYsRows;
  const int nrows = (r0 >= In) ? 0 : (int)((In - r0) < kYsRows ? (In - r0) : kYsRows);
  const bool live = (a.status[0] == 0.0) && nrows > 0;
  // Gamma: its loads are issued before the contraction and consumed after it (unless a Gamma
  // job supplied L^{-1}); warp 0 factors it once the block has it in shared memory
  const bool gjob = (a.linv == nullptr);
  const int CW = gjob ? 7 : 8;  // contraction warps (warp 7 forms and factors Gamma)
  double dfs = 0.0;
  for (int e = tid; e < RR; e += 256) sGram[e] = 0.0;
  if (tid == 0) sfail = 0;
  __syncthreads();
  if (live) {
    const int64_t I0 = a.I0, I1 = a.I1;
    const int64_t blk = I0 * R;  // doubles per i1 slab of Y_L
    if (a.mode == 1 && a.nin > 0) {
      // Upsilon of the new A^(0): the mode-0 kernel's cluster partials, summed in cluster order
      // by all threads (one entry each) before warp 7 forms Gamma from it
      for (int e = tid; e < RR; e += 256) {
        const double u = ys_sum(a.gin + e, RR, a.nin);
        sGram[e] = u;
        if (blockIdx.x == 0) a.Ups[e] = u;
      }
      __syncthreads();
    }
    if (!gjob) {
      for (int e = tid; e < RR; e += 256) sLi[(e / R) * LS + (e % R)] = a.linv[e];
    } else if (warp == 7) {
      ys_gamma_warp<R>(a, sL, sGram, lane);
      __syncwarp();
      ys_chol_warp<R>(sL, sLi, sDi, &sfail, lane);
    }
    YS_T(1);
    // ---- the block's rows of M^(mode) from Y_L (warps < CW) ----
    if (a.mode == 0) {
      // thread (sl, r), sl < nsl: i1 = sl, sl + nsl, ...; the 4 rows i0b.. as one 32-B load when
      // aligned, 8 i1 per batch (16 loads in flight per thread)
      const int nsl = (CW * 32) / R;
      if (tid < nsl * R) {
        const int r = tid % R, sl = tid / R;
        double acc[kYsRows] = {};
        const double *yb = a.yl + (int64_t)r * I0 + r0;
        const double *bt = a.Bfac + r;  // At^(1): row-major, stride RS
        if (nrows == kYsRows && (I0 % kYsRows) == 0) {
          int64_t i1 = sl;
          for (; i1 + 7 * nsl < I1; i1 += 8 * nsl) {
            double y[8][kYsRows], b[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              ld_rows(yb + (i1 + j * nsl) * blk, y[j]);
              b[j] = __ldg(bt + (i1 + j * nsl) * a.RS);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
#pragma unroll
              for (int u = 0; u < kYsRows; ++u) acc[u] = fma(y[j][u], b[j], acc[u]);
          }
          if (i1 < I1) {
            // the remainder as ONE predicated batch (a serial loop here paid one memory round
            // trip per i1: 5 of the 9 round trips of the c4a contraction)
            double y[8][kYsRows], b[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int64_t ij = i1 + j * nsl;
              const int64_t ic = ij < I1 ? ij : (int64_t)sl;
              ld_rows(yb + ic * blk, y[j]);
              b[j] = __ldg(bt + ic * a.RS);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (i1 + j * nsl < I1)
#pragma unroll
                for (int u = 0; u < kYsRows; ++u) acc[u] = fma(y[j][u], b[j], acc[u]);
          }
        } else {
          for (int64_t i1 = sl; i1 < I1; i1 += nsl) {
            const double *yp = yb + i1 * blk;
            const double b = __ldg(bt + i1 * a.RS);
#pragma unroll
            for (int u = 0; u < kYsRows; ++u)
              if (u < nrows) acc[u] = fma(__ldcg(yp + u), b, acc[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < kYsRows; ++u) sP[(sl * R + r) * kYsRows + u] = acc[u];
      }
      __syncthreads();
      if (tid < R * kYsRows) {
        const int r = tid / kYsRows, u = tid % kYsRows;
        double m = 0.0;
        for (int sl = 0; sl < nsl; ++sl) m += sP[(sl * R + r) * kYsRows + u];
        sMv[u * R + r] = m;
      }
    } else if (warp < CW && a.vec1) {
      // warp w owns the ranks r = w, w + CW, ...: for each, the column A^(0)_new(:, r) and the
      // block's Y_L rows (i1 = r0 + u, r) in 32-byte vectors, 2 chunks of 4 x 32 lanes per
      // round trip (A reused over the rows u); lane partials, then a fixed xor tree
      const int64_t nch = I0 / 4;  // 32-B chunks per row
      for (int r = warp; r < R; r += CW) {
        const double *ab = a.Bfac + (int64_t)r * I0;
        const double *yb = a.yl + (int64_t)r * I0 + r0 * blk;
        double acc[kYsRows] = {};
        for (int64_t c0 = lane; c0 < nch; c0 += 64) {
          const int64_t c1 = c0 + 32;
          const bool ok1 = c1 < nch;
          double av[2][4], yv[2][kYsRows][4];
          ld_v4(ab + 4 * c0, av[0]);
          ld_v4(ab + 4 * (ok1 ? c1 : c0), av[1]);
#pragma unroll
          for (int u = 0; u < kYsRows; ++u) {
            const int uc = u < nrows ? u : 0;
            ld_v4(yb + uc * blk + 4 * c0, yv[0][u]);
            ld_v4(yb + uc * blk + 4 * (ok1 ? c1 : c0), yv[1][u]);
          }
#pragma unroll
          for (int u = 0; u < kYsRows; ++u) {
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[u] = fma(yv[0][u][q], av[0][q], acc[u]);
            if (ok1)
#pragma unroll
              for (int q = 0; q < 4; ++q) acc[u] = fma(yv[1][u][q], av[1][q], acc[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < kYsRows; ++u) {
          double t = acc[u];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
          if (lane == 0 && u < nrows) sMv[u * R + r] = t;
        }
      }
    } else if (warp < CW) {
      // warp w owns the entries en = w + CW j (row u = en / R, rank r = en % R) and works on all
      // of them at once; lanes stride i0 (contiguous in Y_L and in the column-major new A^(0)),
      // U chunks of 32 per iteration: EPW * U * 2 loads in flight per lane; fixed xor tree
      constexpr int U = (16 / EPW) > 1 ? (16 / EPW) : 1;
      const int ne = nrows * R;
      int64_t yo[EPW], bo[EPW];
      double acc[EPW];
#pragma unroll
      for (int j = 0; j < EPW; ++j) {
        const int en = warp + CW * j;
        const int enc = en < ne ? en : 0;
        yo[j] = (r0 + enc / R) * blk + (int64_t)(enc % R) * I0;
        bo[j] = (int64_t)(enc % R) * I0;
        acc[j] = 0.0;
      }
      int64_t i0 = lane;
      for (; i0 + 32 * (U - 1) < I0; i0 += 32 * U) {
        double y[U][EPW], b[U][EPW];
#pragma unroll
        for (int c = 0; c < U; ++c)
#pragma unroll
          for (int j = 0; j < EPW; ++j) {
            y[c][j] = __ldcg(a.yl + yo[j] + i0 + 32 * c);
            b[c][j] = __ldg(a.Bfac + bo[j] + i0 + 32 * c);
          }
#pragma unroll
        for (int c = 0; c < U; ++c)
#pragma unroll
          for (int j = 0; j < EPW; ++j) acc[j] = fma(y[c][j], b[c][j], acc[j]);
      }
      for (; i0 < I0; i0 += 32)
#pragma unroll
        for (int j = 0; j < EPW; ++j) acc[j] = fma(__ldcg(a.yl + yo[j] + i0), __ldg(a.Bfac + bo[j] + i0), acc[j]);
#pragma unroll
      for (int j = 0; j < EPW; ++j) {
        double t = acc[j];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        const int en = warp + CW * j;
        if (lane == 0 && en < ne) sMv[en] = t;
      }
    }
    YS_T(6);
    __syncthreads();  // sMv, L^{-1}, sfail complete
    YS_T(2);
    for (int e = tid; e < nrows * R; e += 256) {
      const int u = e / R, r = e % R;
      sB[e] = sMv[e] + (a.F != nullptr ? a.F[(r0 + u) + In * r] : 0.0);
    }
    __syncthreads();
    YS_T(3);
    if (sfail) {
      if (tid == 0) {
        a.status[0] = (double)CP_ENOTSPD;
        a.status[1] = (double)a.mode;
      }
    } else {
      // y = L^{-1} b, x = L^{-T} y; entry e -> (row u fastest, rank r): coalesced A stores
      for (int e = tid; e < nrows * R; e += 256) {
        const int u = e % nrows, r = e / nrows;
        double y = 0.0;
#pragma unroll 4
        for (int k = 0; k <= r; ++k) y = fma(sLi[r * LS + k], sB[u * R + k], y);
        sY[u * R + r] = y;
      }
      __syncthreads();
      double df = 0.0;
      for (int e = tid; e < nrows * R; e += 256) {
        const int u = e % nrows, r = e / nrows;
        double x = 0.0;
#pragma unroll 4
        for (int k = r; k < R; ++k) x = fma(sLi[k * LS + r], sY[u * R + k], x);
        const int64_t i = r0 + u;
        a.A[i + In * r] = x;
        a.At[i * a.RSo + r] = x;
        sX[u * R + r] = x;
        if (a.F != nullptr) df = fma(a.F[i + In * r], x, df);
      }
      // partial Gram of the block's new rows; <F, A> (warp sums in warp order)
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) df += __shfl_xor_sync(0xffffffffu, df, off);
      if (lane == 0) sDot[warp] = df;
      __syncthreads();
      for (int e = tid; e < RR; e += 256) {
        const int r = e % R, s = e / R;
        double gg = 0.0;
        for (int u = 0; u < nrows; ++u) gg = fma(sX[u * R + r], sX[u * R + s], gg);
        sGram[e] = gg;
      }
      if (tid == 0) dfs = ((sDot[0] + sDot[1]) + (sDot[2] + sDot[3])) + ((sDot[4] + sDot[5]) + (sDot[6] + sDot[7]));
    }
  }
  YS_T(4);
  __syncthreads();
  if (tid == 0) sDot[0] = dfs;
  // ---- cluster reduction of the partial Grams and <F, A> (rank order) ----
  cl.sync();
  if (cl.block_rank() == 0) {
    const unsigned cid = blockIdx.x / kYsCluster;
    for (int e = tid; e < RR; e += 256) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < kYsCluster; ++q) s += cl.map_shared_rank(sGram, q)[e];
      a.gcur[(int64_t)cid * RR + e] = s;
    }
    if (tid == 0) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < kYsCluster; ++q) s += cl.map_shared_rank(sDot, q)[0];
      a.dotF[cid] = s;
    }
  }
  cl.sync();  // remote shared memory stays valid until rank 0 has read it
  if (a.total != nullptr && cl.block_rank() == 0) {
    // the last cluster to finish sums the cluster partials (cluster order) into the Gram total
    // of the new factor, so the next kernel reads one value per entry
    __shared__ unsigned sticket;
    __threadfence();
    __syncthreads();
    if (tid == 0) sticket = atomicAdd(a.ticket, 1u);
    __syncthreads();
    const unsigned ncl = gridDim.x / kYsCluster;
    if (sticket == ncl - 1) {
      __threadfence();
      for (int e = tid; e < RR; e += 256) a.total[e] = ys_sum(a.gcur + e, RR, (int)ncl);
      if (tid == 0) *a.ticket = 0u;
    }
  }
  YS_T(5);
  CTL_END(a.mode == 0 ? "ylsolve0" : "ylsolve1")
#ifdef CP_SOLVE_TIMING
  if (threadIdx.x == 0)
    printf("YS %d %d %llu %llu %llu %llu %llu %llu %llu %llu\n", a.mode, blockIdx.x, tst[0], tst[1], tst[6], tst[7], tst[2], tst[3], tst[4], tst[5]);
#endif
}

int ylsolve_clusters(int64_t In) {
  const int64_t blocks = (In + kYsRows - 1) / kYsRows;
  return (int)((blocks + kYsCluster - 1) / kYsCluster);
}

template <int R>
static cudaError_t launch_ylsolve_t(const YLSolveArgs &a, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ylsolve_clusters(a.In) * kYsCluster));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled(kPdlCluster) ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ylsolve_kernel_t<R>, a);
}

cudaError_t launch_ylsolve(const YLSolveArgs &a, cudaStream_t st) {
  switch (a.R) {
#define CPK_YS_CASE(r) \
  case r: return launch_ylsolve_t<r>(a, st);
    CPK_YS_CASE(1) CPK_YS_CASE(2) CPK_YS_CASE(3) CPK_YS_CASE(4) CPK_YS_CASE(5) CPK_YS_CASE(6) CPK_YS_CASE(7)
    CPK_YS_CASE(8) CPK_YS_CASE(9) CPK_YS_CASE(10) CPK_YS_CASE(11) CPK_YS_CASE(12) CPK_YS_CASE(13)
    CPK_YS_CASE(14) CPK_YS_CASE(15) CPK_YS_CASE(16) CPK_YS_CASE(17) CPK_YS_CASE(18) CPK_YS_CASE(19)
    CPK_YS_CASE(20) CPK_YS_CASE(21) CPK_YS_CASE(22) CPK_YS_CASE(23) CPK_YS_CASE(24) CPK_YS_CASE(25)
    CPK_YS_CASE(26) CPK_YS_CASE(27) CPK_YS_CASE(28) CPK_YS_CASE(29) CPK_YS_CASE(30) CPK_YS_CASE(31)
    CPK_YS_CASE(32)
#undef CPK_YS_CASE
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace cpk
