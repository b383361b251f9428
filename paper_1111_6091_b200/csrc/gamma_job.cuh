// gamma_job.cuh -- Gamma^(n) = *_{k != n} Upsilon^(k) (eq:Gamma) and the inverse of its
// Cholesky factor, L^{-1} (reading R1), computed off the solve's critical path.
//
// In the dimension-tree sweep each Gamma^(n) depends only on Grams that exist one kernel
// earlier than the solve of mode n, so a "job" rides along in that earlier kernel: the idle
// weight warp of a streaming kernel (one warp of CTA 0) or one extra block of a Y_L / Y_R
// contraction kernel.  The job sums the Gram partials it is given in fixed order (writing the
// totals to Ups), forms Gamma in shared memory, factors it right-looking (no pivoting; a
// non-positive or NaN pivot reports CP_ENOTSPD for the mode; 1/L(j,j) = rsqrt(pivot)) and
// writes L^{-1} (row-major, R x R, lower) by forward substitution, one column per thread.
// The solve kernel then only reads L^{-1}.  Runtime R (no per-R instantiations).
#pragma once
#include "cp_internal.cuh"

namespace cpk {

// doubles of shared memory a job needs (R x (R + 1) matrix + R diagonal inverses + flag)
__host__ __device__ constexpr int gamma_job_smem_doubles(int R) { return R * (R + 1) + R + 2; }

// sum of n values at stride, 8 loads in flight, fixed combination order
__device__ __forceinline__ double gj_sum(const double *p, int64_t stride, int n) {
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

// Run the job with threads t = 0..nthr-1 of the caller (one warp, block = false, or a whole
// block, block = true); every one of them calls it.  sg: gamma_job_smem_doubles(R) doubles.
static __device__ __noinline__ void gamma_job_run(const GammaJob &g, double *sg, int t, int nthr, bool block) {
  if (g.status[0] != 0.0) return;  // an earlier mode already failed (uniform for the caller)
  const int R = g.R, RR = R * R, LS = R + 1;
  double *sd = sg + R * LS;                          // 1 / L(j, j)
  volatile double *sflag = sd + R;                    // 0: ok, 1: not SPD
  auto sync = [&]() {
    if (block) __syncthreads();
    else __syncwarp();
  };
  for (int e = t; e < RR; e += nthr) {
    double gm = 1.0;
    for (int k = 0; k < g.N; ++k) {
      if (k == g.mode) continue;
      double u;
      if (g.cnt[k] > 0) {
        u = gj_sum(g.src[k] + e, RR, g.cnt[k]);
        g.ups[(int64_t)k * RR + e] = u;
      } else {
        u = g.src[k][e];
      }
      gm *= u;
    }
    sg[(e % R) * LS + e / R] = gm;
  }
  if (t == 0) sflag[0] = 0.0;
  sync();
  // right-looking Cholesky of the lower triangle
  for (int j = 0; j < R; ++j) {
    if (t == 0) {
      const double piv = sg[j * LS + j];
      if (!(piv > 0.0)) {
        sflag[0] = 1.0;
      } else {
        const double inv = rsqrt(piv);
        sd[j] = inv;
        sg[j * LS + j] = piv * inv;
      }
    }
    sync();
    if (sflag[0] != 0.0) break;
    const double inv = sd[j];
    for (int i = j + 1 + t; i < R; i += nthr) sg[i * LS + j] *= inv;
    sync();
    const int m = R - j - 1;
    for (int e = t; e < m * m; e += nthr) {
      const int i = j + 1 + e / m, k = j + 1 + e % m;
      if (k <= i) sg[i * LS + k] = fma(-sg[i * LS + j], sg[k * LS + j], sg[i * LS + k]);
    }
    sync();
  }
  if (sflag[0] != 0.0) {
    if (t == 0) {
      g.status[0] = (double)CP_ENOTSPD;
      g.status[1] = (double)g.mode;
    }
    return;
  }
  // L^{-1}: thread c forms column c by forward substitution; x_i (i >= c) is kept in row c of
  // sg at and right of the diagonal, which the substitution never reads as L (it reads the
  // strictly lower triangle and sd)
  for (int c = t; c < R; c += nthr) {
    for (int i = c; i < R; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) s = fma(-sg[i * LS + k], sg[c * LS + k], s);
      sg[c * LS + i] = s * sd[i];
    }
    for (int i = 0; i < R; ++i) g.linv[i * R + c] = (i >= c) ? sg[c * LS + i] : 0.0;
  }
}

}  // namespace cpk
