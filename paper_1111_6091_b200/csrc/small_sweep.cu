// Fused ALS / BNGS sweeps for a tensor that fits in one CTA's shared memory (the coarse levels of
// the multigrid hierarchy: c1 50^3 -> 25^3 -> 13^3 -> 7^3 -> 4^3).
//
// The coarsest level runs nu_c = 50 relaxation sweeps per V-cycle (Table 1).  On the
// general path a sweep is ~8 launches whose work is a few hundred flops each at 4^3, so the
// V-cycle is launch-latency bound.  Here ONE launch runs `nsweeps` complete sweeps (for
// n = 1..N, M = Z_(n)Phi^(n) (eq:gradEqn), Gamma = *_{k != n} A^(k)T A^(k) (eq:Gamma),
// A^(n) Gamma = M + F (eq:relaxinnersolve P:356-358) by Cholesky) with Z, every factor and every
// Gram resident in shared memory, and returns f, f~ after the last sweep exactly as
// cp_als_sweep does (readings R5, R6).  Every sum has a fixed order: bitwise reproducible.
#include <cstdio>

#include "cp_internal.cuh"
#include "small_sweep.cuh"

namespace cpk {

#ifdef CP_SMALL_TIMING
#define ST(k) if (threadIdx.x == 0 && sweep == 1) tst[k] = clock64();
#else
#define ST(k)
#endif

namespace {
constexpr int kT = kSmallSweepThreads;
// smallest R whose Cholesky runs on warp 0 (tools/chol_ab.py: R = 3 one thread 12.4 us/sweep vs
// warp 12.9 at 4^3; R = 8 34.5 vs 30.2 at 7^3; R = 32 450 vs 209 at 13^3)
constexpr int kSmallCholWarpMinR = 5;
// R <= this: warp 0 factors Gamma with its rows in registers (shuffles; round 2) instead of the
// one-thread loop; R = 5..8 keep the warp loop below (the register variant measured 5 % slower
// at 7^3 R = 8)
constexpr int kSmallCholRegMaxR = 4;

// 1/sqrt(x), x > 0: rsqrt.approx.f64 + two Newton steps (as ys_rsqrt in ylsolve.cu): no
// square root or division on the serial Cholesky chain
__device__ __forceinline__ double ss_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx, y * y, 1.5);
  y = y * fma(-hx, y * y, 1.5);
  return y;
}

// x / d for 0 <= x < 2^22, d >= 1, from a float reciprocal plus one correction (exact): the
// hardware has no integer divider, and the generic 32-bit division sequence dominated the tiny
// phases of this kernel
__device__ __forceinline__ int qdiv(int x, int d, float inv) {
  int q = __float2int_rz((float)x * inv);
  const int r = x - q * d;
  q += (r >= d) - (r < 0);
  return q;
}

// fixed-order block sum of one value per thread (red: KT doubles); result in every thread
template <int KT>
__device__ double block_sum_fixed(double v, double *red) {
  const int tid = threadIdx.x;
  __syncthreads();
  red[tid] = v;
  __syncthreads();
  for (int off = KT / 2; off > 0; off >>= 1) {
    if (tid < off) red[tid] += red[tid + off];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}
}  // namespace

// KT threads (512; a 128-thread instance for 4^3 / 7^3 measured 7-27 % slower)
template <int KT>
__global__ void __launch_bounds__(KT) small_sweep_kernel(const SmallSweepArgs a) {
  griddep();
  extern __shared__ double sm[];
  const int tid = threadIdx.x, N = a.N, R = a.R, RR = R * R;
  const float inv_R = 1.0f / (float)R;
  const int64_t P = a.P;
  // shared layout (doubles): Z | A^(0..N-1) | Ups^(0..N-1) | M | part | WL | WR | Gam | L | red
  double *sZ = sm;
  // factor offsets and dims in shared memory (dynamically indexed: no local-memory copies)
  __shared__ int s_aoff[CP_MAX_N], s_dims[CP_MAX_N];
  __shared__ float s_inv[CP_MAX_N];
  int64_t off = P;
  for (int k = 0; k < N; ++k) {
    if (tid == 0) {
      s_aoff[k] = (int)off;
      s_dims[k] = (int)a.dims[k];
      s_inv[k] = 1.0f / (float)a.dims[k];
    }
    off += a.dims[k] * R;
  }
  double *sU = sm + off;
  off += (int64_t)N * RR;
  double *sM = sm + off;
  off += a.imax * R;
  double *part = sm + off;
  off += a.npart + a.lr * R;  // part | WL | WR
  double *sG = sm + off;
  off += RR;
  double *sL = sm + off;
  off += RR;
  double *red = sm + off;
  __shared__ int s_status, s_failed;
  __shared__ double sDi[kSmallSweepMaxR];  // 1 / L(r, r)

  __syncthreads();
  for (int64_t e = tid; e < P; e += KT) sZ[e] = a.Z[e];
  for (int k = 0; k < N; ++k)
    for (int64_t e = tid; e < s_dims[k] * R; e += KT) (sm + s_aoff[k])[e] = a.A[k][e];
  if (tid == 0) {
    s_status = 0;
    s_failed = -1;
  }
  __syncthreads();
  // Upsilon^(k) = A^(k)T A^(k), sum over i ascending
  for (int e = tid; e < N * RR; e += KT) {
    const int k = e / RR, rs = e - k * RR, r = rs % R, s = rs / R;
    const double *x = (sm + s_aoff[k]) + s_dims[k] * r, *y = (sm + s_aoff[k]) + s_dims[k] * s;
    double g = 0.0;
    for (int64_t i = 0; i < s_dims[k]; ++i) g = fma(x[i], y[i], g);
    sU[e] = g;
  }
  __syncthreads();

  double inner_last = 0.0, inner_grad = 0.0, gsum = 0.0, model2_last = 0.0, fa_last = 0.0;
  // passes: the nsweeps sweeps, then (grad_after) one gradient pass at the new iterate; pure
  // gradient mode (a.grad) is that pass alone
  const int npass = a.grad ? 1 : a.nsweeps + (a.grad_after ? 1 : 0);
#ifdef CP_SMALL_TIMING
  long long tst[16] = {0};
#endif
  for (int sweep = 0; sweep < npass && s_status == 0; ++sweep) {
    const bool gpass = a.grad || sweep == a.nsweeps;
    for (int n = 0; n < N; ++n) {
      // Z viewed as left x I_n x right (left = prod_{k<n} I_k); the Khatri-Rao row of column
      // (a, b) is WL(a, :) * WR(b, :) with WL = the left modes' rows (P:110 order), WR the right
      if (n == 0) ST(0);
      const int In = (int)s_dims[n];
      int left = 1, right = 1;
      for (int k = 0; k < n; ++k) left *= (int)s_dims[k];
      for (int k = n + 1; k < N; ++k) right *= (int)s_dims[k];
      double *sWL = part + a.npart, *sWR = sWL + (int64_t)left * R;
      const float inv_left = 1.0f / (float)left, inv_right = 1.0f / (float)right, inv_In = s_inv[n];
      for (int e = tid; e < (left + right) * R; e += KT) {
        const bool isl = e < left * R;
        const int ee = isl ? e : e - left * R;
        const int len = isl ? left : right;
        const int r = qdiv(ee, len, isl ? inv_left : inv_right);
        int c = ee - r * len;
        double w = 1.0;
        for (int k = isl ? 0 : n + 1; k < (isl ? n : N); ++k) {
          const int Ik = (int)s_dims[k];
          const int c2 = qdiv(c, Ik, s_inv[k]);
          const int ik = c - c2 * Ik;
          c = c2;
          w *= (sm + s_aoff[k])[ik + Ik * r];
        }
        (isl ? sWL : sWR)[ee] = w;  // ee = c + len * r
      }
      __syncthreads();
      if (n == 0) ST(1);
      // ---- M(i, r) = sum_{a,b} z(a, i, b) WL(a, r) WR(b, r) (eq:gradEqn): a warp per output
      // entry, its lanes stride over the columns q = a + left b, fixed xor-tree reduction ----
      const int Q = left * right;
      const int nout = In * R;
      {
        const int warp = tid >> 5, lane = tid & 31;
        const int bstride = left * In;
        for (int o = warp; o < nout; o += KT / 32) {
          const int r = qdiv(o, In, inv_In), i = o - r * In;
          const double *wl = sWL + left * r, *wr = sWR + right * r;
          const double *zrow = sZ + left * i;
          double acc = 0.0;
          if (left == 1) {
            const double w0 = wl[0];
            for (int q = lane; q < Q; q += 32) acc = fma(zrow[bstride * q], w0 * wr[q], acc);
          } else if (right == 1) {
            const double w0 = wr[0];
            for (int q = lane; q < Q; q += 32) acc = fma(zrow[q], wl[q] * w0, acc);
          } else {
            for (int q = lane; q < Q; q += 32) {
              const int bb = qdiv(q, left, inv_left), aa = q - bb * left;
              acc = fma(zrow[aa + bstride * bb], wl[aa] * wr[bb], acc);
            }
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
          if (lane == 0) sM[o] = acc;
        }
      }
      __syncthreads();
      if (n == 0) ST(2);
      // Gamma^(n) = *_{k != n} Upsilon^(k) (eq:Gamma)
      for (int e = tid; e < RR; e += KT) {
        double g = 1.0;
        for (int k = 0; k < N; ++k)
          if (k != n) g *= sU[k * RR + e];
        sG[e] = g;
      }
      __syncthreads();
      if (n == 0) ST(3);
      if (gpass) {
        // ---- cp_gradient: G = -M + A Gamma - F at this iterate (eq:gradEqn), ||G||^2 ----
        const double *Fg = a.gF[n];
        double *G = a.G[n];
        const double *An = sm + s_aoff[n];
        double g2 = 0.0, d = 0.0;
        for (int o = tid; o < nout; o += KT) {
          const int r = qdiv(o, In, inv_In), i = o - r * In;
          double gv = -sM[o];
          for (int t = 0; t < R; ++t) gv = fma(An[i + In * t], sG[t + R * r], gv);
          if (Fg != nullptr) gv -= Fg[o];
          if (G != nullptr) G[o] = gv;
          g2 = fma(gv, gv, g2);
          if (n == N - 1) d = fma(sM[o], An[o], d);
        }
        const double g2s = block_sum_fixed<KT>(g2, red);
        if (tid == 0) a.gout[2 + n] = g2s;
        gsum += g2s;
        if (n == N - 1) inner_grad = block_sum_fixed<KT>(d, red);
        continue;
      }
      // ---- Gamma = L L^T, lower, no pivoting; pivot <= 0 -> CP_ENOTSPD ----
      // R <= 4: one thread (the serial chain is short; measured faster).  Otherwise:
      // Column j by warp 0, lane i = row i (R <= 32): each lane forms its own
      //   s_i = Gamma(i,j) - sum_{k<j} L(i,k) L(j,k)
      // in the same order and expression the former one-thread loop used (bitwise identical
      // L), so the serial chain per column is j multiply-adds instead of (R - j) * j.
      if (R <= kSmallCholRegMaxR) {
        // R <= 8: warp 0 with the rows in registers (lane i = row i), pivots by shuffle -- the
        // one-thread loop below made every step a dependent shared-memory round trip (~2 k
        // cycles per mode at R = 3, CP_SMALL_TIMING)
        if (tid < 32) {
          const int lane = tid;
          constexpr int MR = kSmallCholRegMaxR;
          double g[MR];
#pragma unroll
          for (int c = 0; c < MR; ++c) g[c] = (lane < R && c < R) ? sG[lane + R * c] : 0.0;
          bool okc = true;
#pragma unroll
          for (int j = 0; j < MR; ++j) {
            if (j < R) {
              const double piv = __shfl_sync(0xffffffffu, g[j], j);
              okc = okc && (piv > 0.0);
              const double inv = ss_rsqrt(okc ? piv : 1.0);
              if (lane == 0) sDi[j] = inv;
              if (lane == j) g[j] = piv * inv;
              else if (lane > j) g[j] *= inv;
#pragma unroll
              for (int k = j + 1; k < MR; ++k) {
                const double lkj = __shfl_sync(0xffffffffu, g[j], k);
                if (k < R && lane >= k) g[k] = fma(-g[j], lkj, g[k]);
              }
            }
          }
          if (!okc) {
            if (lane == 0) {
              s_status = CP_ENOTSPD;
              s_failed = n;
            }
          } else if (lane < R) {
#pragma unroll
            for (int c = 0; c < MR; ++c)
              if (c < R) sL[lane + R * c] = (c <= lane) ? g[c] : 0.0;
          }
        }
      } else if (R < kSmallCholWarpMinR) {
        if (tid == 0) {
          for (int e = 0; e < RR; ++e) sL[e] = 0.0;
          for (int j = 0; j < R && s_status == 0; ++j) {
            double d = sG[j + R * j];
            for (int k = 0; k < j; ++k) d -= sL[j + R * k] * sL[j + R * k];
            if (!(d > 0.0)) {
              s_status = CP_ENOTSPD;
              s_failed = n;
              break;
            }
            const double rj = ss_rsqrt(d), ljj = d * rj;
            sL[j + R * j] = ljj;
            sDi[j] = rj;
            for (int i = j + 1; i < R; ++i) {
              double s = sG[i + R * j];
              for (int k = 0; k < j; ++k) s -= sL[i + R * k] * sL[j + R * k];
              sL[i + R * j] = s * rj;
            }
          }
        }
      } else if (tid < 32) {
        const int lane = tid;
        for (int e = lane; e < RR; e += 32) sL[e] = 0.0;
        __syncwarp();
        for (int j = 0; j < R; ++j) {
          // every lane also forms the pivot itself (same order: the lane-j value), no shuffle
          double s = 0.0, d = sG[j + R * j];
          for (int k = 0; k < j; ++k) d -= sL[j + R * k] * sL[j + R * k];
          if (lane > j && lane < R) {
            s = sG[lane + R * j];
            for (int k = 0; k < j; ++k) s -= sL[lane + R * k] * sL[j + R * k];
          }
          if (!(d > 0.0)) {
            if (lane == 0) {
              s_status = CP_ENOTSPD;
              s_failed = n;
            }
            break;
          }
          const double rj = ss_rsqrt(d);
          if (lane == j) {
            sL[j + R * j] = d * rj;  // lane j's s is d
            sDi[j] = rj;
          } else if (lane > j && lane < R) {
            sL[lane + R * j] = s * rj;
          }
          __syncwarp();
        }
      }
      __syncthreads();
      if (n == 0) ST(4);
      if (s_status != 0) break;
      // ---- each row: L y = (m + f)^T, L^T x^T = y (eq:relaxinnersolve) ----
      const double *F = a.F[n];
      __syncthreads();  // (part is reused for y below)
      if (R >= kSmallCholWarpMinR) {
        // one warp per row, lane r = component r.  Forward: column-oriented (after y_r, lanes
        // k > r subtract L(k,r) y_r) -- each b_k sees the subtractions in the same order
        // k' = 0..k-1 as the row-oriented loop below, so y is bitwise the same.  Backward:
        // lane j subtracts L(r,j) x_r for r = R-1 down to j+1 (the reverse of the row loop's
        // order; a rounding-level difference).  The serial chain per row is 2R shuffles+FMAs
        // instead of R^2 dependent shared-memory FMAs (13^3 R = 32: 51 k -> see DESIGN 6.7).
        const int lane = tid & 31, warp = tid >> 5;
        double *An = sm + s_aoff[n];
        const double dl = lane < R ? sDi[lane] : 0.0;
        for (int i = warp; i < In; i += KT / 32) {
          double b = 0.0;
          if (lane < R) b = sM[i + In * lane] + (F != nullptr ? F[i + In * lane] : 0.0);
          for (int r = 0; r < R; ++r) {
            const double yr = __shfl_sync(0xffffffffu, b * dl, r);
            if (lane == r) b = yr;
            else if (lane > r && lane < R) b -= sL[lane + R * r] * yr;
          }
          for (int r = R - 1; r >= 0; --r) {
            const double xr = __shfl_sync(0xffffffffu, b * dl, r);
            if (lane == r) b = xr;
            else if (lane < r) b -= sL[r + R * lane] * xr;
          }
          if (lane < R) An[i + In * lane] = b;
        }
      } else
      for (int i = tid; i < In; i += KT) {
        // R < 5: a thread per row with the row in registers (the loads of a step are independent)
        constexpr int MR = kSmallCholWarpMinR - 1;
        double y[MR];
#pragma unroll
        for (int r = 0; r < MR; ++r)
          if (r < R) y[r] = sM[i + In * r] + (F != nullptr ? F[i + In * r] : 0.0);
#pragma unroll
        for (int r = 0; r < MR; ++r) {
          if (r < R) {
            double b = y[r];
#pragma unroll
            for (int k = 0; k < r; ++k) b -= sL[r + R * k] * y[k];
            y[r] = b * sDi[r];
          }
        }
#pragma unroll
        for (int r = MR - 1; r >= 0; --r) {
          if (r < R) {
            double x = y[r];
#pragma unroll
            for (int k = r + 1; k < MR; ++k)
              if (k < R) x -= sL[k + R * r] * y[k];
            y[r] = x * sDi[r];
            (sm + s_aoff[n])[i + In * r] = y[r];
          }
        }
      }
      __syncthreads();
      if (n == 0) ST(5);
      // Upsilon^(n) of the new factor
      for (int e = tid; e < RR; e += KT) {
        const int s = qdiv(e, R, inv_R), r = e - s * R;
        const double *x = (sm + s_aoff[n]) + In * r, *y = (sm + s_aoff[n]) + In * s;
        double g = 0.0;
        for (int i = 0; i < In; ++i) g = fma(x[i], y[i], g);
        sU[n * RR + e] = g;
      }
      if (n == N - 1 && sweep == a.nsweeps - 1) {
        double d = 0.0;
        for (int o = tid; o < nout; o += KT) d = fma(sM[o], (sm + s_aoff[n])[o], d);
        inner_last = block_sum_fixed<KT>(d, red);
      }
      __syncthreads();
      if (n == 0) ST(6);
    }
    if (gpass || s_status != 0) continue;
    if (sweep == a.nsweeps - 1) {
      // f pieces of the last sweep, before any normalization (as cp_als_sweep then
      // cp_normalize_sort): ||[[A]]||^2 = 1^T (*_k Upsilon^(k)) 1 and sum_n <F^(n), A^(n)>
      double m2 = 0.0;
      for (int e = tid; e < RR; e += KT) {
        double p = 1.0;
        for (int k = 0; k < N; ++k) p *= sU[k * RR + e];
        m2 += p;
      }
      model2_last = block_sum_fixed<KT>(m2, red);
      double fa = 0.0;
      for (int k = 0; k < N; ++k)
        if (a.F[k] != nullptr)
          for (int64_t e = tid; e < s_dims[k] * R; e += KT) fa = fma(a.F[k][e], (sm + s_aoff[k])[e], fa);
      fa_last = block_sum_fixed<KT>(fa, red);
    }
    if (a.normalize) {
      // eq:ALSnorm after the sweep (cp_normalize_sort with sort = 0): every column
      // scaled to lambda_r = (prod_n ||a_r^(n)||)^(1/N), unless a column norm is zero
      __shared__ double sNrm[CP_MAX_N * kSmallSweepMaxR], sLam[kSmallSweepMaxR];
      __shared__ int sPos[kSmallSweepMaxR];
      for (int e = tid; e < N * R; e += KT) {
        const int k = e / R, r = e - k * R;
        const double *col = (sm + s_aoff[k]) + s_dims[k] * r;
        double ss = 0.0;
        for (int i = 0; i < s_dims[k]; ++i) ss = fma(col[i], col[i], ss);
        sNrm[e] = sqrt(ss);
      }
      __syncthreads();
      for (int r = tid; r < R; r += KT) {
        double prod = 1.0;
        int pos = 1;
        for (int k = 0; k < N; ++k) {
          prod *= sNrm[k * R + r];
          pos = pos && (sNrm[k * R + r] > 0.0);
        }
        sLam[r] = pow(prod, 1.0 / (double)N);
        sPos[r] = pos;
      }
      __syncthreads();
      for (int k = 0; k < N; ++k) {
        double *Ak = sm + s_aoff[k];
        for (int e = tid; e < s_dims[k] * R; e += KT) {
          const int r = e / s_dims[k];
          if (sPos[r]) Ak[e] = sLam[r] * (Ak[e] / sNrm[k * R + r]);
        }
      }
      __syncthreads();
      for (int e = tid; e < N * RR; e += KT) {  // the Grams of the normalized factors
        const int k = e / RR, rs = e - k * RR, r = rs % R, s2 = rs / R;
        const double *x = (sm + s_aoff[k]) + s_dims[k] * r, *y = (sm + s_aoff[k]) + s_dims[k] * s2;
        double g = 0.0;
        for (int i = 0; i < s_dims[k]; ++i) g = fma(x[i], y[i], g);
        sU[e] = g;
      }
      __syncthreads();
    }
  }

#ifdef CP_SMALL_TIMING
  if (threadIdx.x == 0)
    printf("small sweep phases (clk, mode 0 of sweep 1): wlwr %lld mttkrp %lld msum+gamma %lld chol %lld solve %lld gram %lld\n",
           tst[1] - tst[0], tst[2] - tst[1], tst[3] - tst[2], tst[4] - tst[3], tst[5] - tst[4], tst[6] - tst[5]);
#endif
  if (a.grad || (a.grad_after && s_status == 0)) {
    // f by the expansion (reading R6), g = (sum_n ||G^(n)||^2)^{1/2} / ||Z|| (eq:gradConv)
    double m2 = 0.0;
    for (int e = tid; e < RR; e += KT) {
      double p = 1.0;
      for (int k = 0; k < N; ++k) p *= sU[k * RR + e];
      m2 += p;
    }
    const double model2 = block_sum_fixed<KT>(m2, red);
    if (tid == 0) {
      a.gout[0] = 0.5 * a.normZ2[0] - inner_grad + 0.5 * model2;
      a.gout[1] = sqrt(gsum) / sqrt(a.normZ2[0]);
    }
    if (a.grad) return;
  } else if (a.grad_after && tid == 0) {
    a.gout[0] = nan("");  // the sweeps failed (CP_ENOTSPD in out): no gradient
    a.gout[1] = nan("");
  }
  // ---- write back, f and f~ (readings R6, R5) ----
  for (int k = 0; k < N; ++k)
    for (int64_t e = tid; e < s_dims[k] * R; e += KT) a.A[k][e] = (sm + s_aoff[k])[e];
  if (s_status != 0) {
    if (tid == 0) {
      a.out[0] = nan("");
      a.out[1] = nan("");
      a.out[2] = (double)s_status;
      a.out[3] = (double)s_failed;
    }
    return;
  }
  const double model2 = model2_last, fas = fa_last;
  if (tid == 0) {
    const double f = 0.5 * a.normZ2[0] - inner_last + 0.5 * model2;
    a.out[0] = f;
    a.out[1] = f - fas;
    a.out[2] = 0.0;
    a.out[3] = -1.0;
  }
}

size_t small_sweep_smem_bytes(const cp_shape &s) {
  if (s.R > kSmallSweepMaxR) return 0;
  double P = 1.0;
  int64_t imax = 1, sumI = 0;
  for (int k = 0; k < s.N; ++k) {
    P *= (double)s.dims[k];
    sumI += s.dims[k];
    if (s.dims[k] > imax) imax = s.dims[k];
  }
  if (P > (double)kSmallSweepMaxP) return 0;
  const int64_t npart = imax * s.R > kT ? imax * s.R : kT;
  double lr = 0.0;  // Khatri-Rao halves WL, WR of the largest mode geometry
  for (int n = 0; n < s.N; ++n) {
    double left = 1.0, right = 1.0;
    for (int k = 0; k < n; ++k) left *= (double)s.dims[k];
    for (int k = n + 1; k < s.N; ++k) right *= (double)s.dims[k];
    if (left + right > lr) lr = left + right;
  }
  const double d = P + (double)sumI * s.R + (double)s.N * s.R * s.R + (double)imax * s.R + (double)npart +
                   lr * s.R + 2.0 * s.R * s.R + kT;
  return (size_t)(d * 8.0);
}

cudaError_t launch_small_sweep(const cp_shape &s, const double *Z, const double *normZ2, double *const *A,
                               const double *const *F, int nsweeps, double *out, cudaStream_t st,
                               double *const *G, bool grad, bool normalize, double *gout,
                               const double *const *gF) {
  SmallSweepArgs a;
  memset(&a, 0, sizeof(a));
  a.grad = grad ? 1 : 0;
  a.normalize = normalize ? 1 : 0;
  // pure gradient mode: F enters G, results in out; sweeps + gradient: separate F / outputs
  a.grad_after = (!grad && gout != nullptr) ? 1 : 0;
  a.gout = grad ? out : gout;
  for (int k = 0; k < s.N; ++k) {
    a.G[k] = (G != nullptr) ? G[k] : nullptr;
    a.gF[k] = grad ? ((F != nullptr) ? F[k] : nullptr) : ((gF != nullptr) ? gF[k] : nullptr);
  }
  a.N = s.N;
  a.R = s.R;
  a.nsweeps = nsweeps;
  a.P = 1;
  a.imax = 1;
  for (int k = 0; k < s.N; ++k) {
    a.dims[k] = s.dims[k];
    a.P *= s.dims[k];
    if (s.dims[k] > a.imax) a.imax = s.dims[k];
    a.A[k] = const_cast<double *>(A[k]);
    a.F[k] = (F != nullptr) ? F[k] : nullptr;
  }
  a.npart = a.imax * s.R > kT ? a.imax * s.R : kT;
  a.lr = 0;
  for (int n = 0; n < s.N; ++n) {
    int64_t left = 1, right = 1;
    for (int k = 0; k < n; ++k) left *= s.dims[k];
    for (int k = n + 1; k < s.N; ++k) right *= s.dims[k];
    if (left + right > a.lr) a.lr = left + right;
  }
  a.Z = Z;
  a.normZ2 = normZ2;
  a.out = out;
  const size_t smem = small_sweep_smem_bytes(s);
  if (smem > 48 * 1024) {
    cudaError_t e = ensure_smem_attr((const void *)small_sweep_kernel<kT>, (int)smem);
    if (e != cudaSuccess) return e;
  }
  return launch_k(small_sweep_kernel<kT>, dim3(1), dim3(kT), smem, st, a);
}

}  // namespace cpk
