// small_kernels.cu -- the R x R side of the hot path (eq:Gamma P:113-116, Cholesky solve of
// P:121 / eq:relaxinnersolve P:356-358, the functional eq:CPfunctional P:38-42, the gradient
// eq:gradEqn and g eq:gradConv P:454-456) plus ||Z||^2.  All reductions run in a fixed order
// (no atomics), so results are bitwise reproducible.
#include "small_kernels.cuh"

namespace cpk {

// ---------------------------------------------------------------- reduction of stream partials
__device__ __forceinline__ double reduce_entry(const ReduceGeom &g, int64_t i, int r) {
  double s = 0.0;
  if (g.mode0) {  // mode 0: one I1 x R partial per column group
    const double *p = g.part + i + g.I1 * r;
    const int64_t stride = g.I1 * g.R;
    int c = 0;
    double s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (; c + 3 < g.Gc; c += 4) {  // four independent chains, combined in fixed order
      s += p[(int64_t)c * stride];
      s1 += p[(int64_t)(c + 1) * stride];
      s2 += p[(int64_t)(c + 2) * stride];
      s3 += p[(int64_t)(c + 3) * stride];
    }
    for (; c < g.Gc; ++c) s += p[(int64_t)c * stride];
    s = (s + s1) + (s2 + s3);
  } else {  // mode m >= 1: R-vector partials per (column group, row block, segment)
    const int64_t lo = i * g.Qn, hi = (i + 1) * g.Qn - 1;
    const int64_t clo = ((lo + 1) * g.Gc - 1) / g.Q;
    const int64_t chi = ((hi + 1) * g.Gc - 1) / g.Q;
    for (int64_t c = clo; c <= chi; ++c) {
      const int64_t seg_first = ((c * g.Q) / g.Gc) / g.Qn;
      for (int rb = 0; rb < g.RB; ++rb)
        s += g.part[(((c * g.RB + rb) * g.slots) + (i - seg_first)) * g.R + r];
    }
  }
  return s;
}

__global__ void reduce_mttkrp_kernel(const ReduceGeom g, double *M) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= g.In_rows * g.R) return;
  const int64_t i = idx % g.In_rows;
  const int r = (int)(idx / g.In_rows);
  M[i + g.In_rows * r] = reduce_entry(g, i, r);
}

// ---------------------------------------------------------------- prep: At copies + Grams
// block k: At^(k) (row-major copy), Upsilon^(k) = A^(k)^T A^(k), fixed-order sums.
__global__ void prep_kernel(const PrepArgs a) {
  const int k = blockIdx.x;
  const int R = a.R;
  const int64_t I = a.dims[k];
  const double *A = a.A[k];
  if (A == nullptr) return;
  double *At = a.At[k];
  const int RS = R + (R & 1);  // padded row stride (16-B aligned rows for the TMA copies)
  for (int64_t e = threadIdx.x; e < I * RS; e += blockDim.x) {
    const int64_t i = e / RS;
    const int r = (int)(e - i * RS);
    At[e] = (r < R) ? A[i + I * r] : 0.0;
  }
  if (a.Ups != nullptr) {
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      const int r = e % R, s = e / R;
      const double *ar = A + I * r;
      const double *as = A + I * s;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int64_t i = 0;
      for (; i + 3 < I; i += 4) {
        s0 = fma(ar[i], as[i], s0);
        s1 = fma(ar[i + 1], as[i + 1], s1);
        s2 = fma(ar[i + 2], as[i + 2], s2);
        s3 = fma(ar[i + 3], as[i + 3], s3);
      }
      for (; i < I; ++i) s0 = fma(ar[i], as[i], s0);
      a.Ups[(int64_t)k * R * R + e] = (s0 + s1) + (s2 + s3);
    }
  }
  if (k == 0 && threadIdx.x == 0 && a.status != nullptr) {
    a.status[0] = 0.0;
    a.status[1] = -1.0;
  }
}

// Cholesky Gamma = L L^T (lower, no pivoting) of an R x R matrix in shared memory (stride 33),
// by one warp: lane i owns row i.  Returns false on a pivot <= 0 (or NaN).
__device__ bool warp_cholesky(double *G, int R, int lane) {
  bool ok = true;
  for (int j = 0; j < R; ++j) {
    double d = 0.0;
    if (lane == j) {
      d = G[j * 33 + j];
      for (int k = 0; k < j; ++k) d -= G[j * 33 + k] * G[j * 33 + k];
    }
    d = __shfl_sync(0xffffffffu, d, j);
    if (!(d > 0.0)) {
      ok = false;
      break;
    }
    const double ljj = sqrt(d);
    if (lane == j) G[j * 33 + j] = ljj;
    __syncwarp();
    if (lane > j && lane < R) {
      double s = G[lane * 33 + j];
      for (int k = 0; k < j; ++k) s -= G[lane * 33 + k] * G[j * 33 + k];
      G[lane * 33 + j] = s / ljj;
    }
    __syncwarp();
  }
  return ok;
}

// ---------------------------------------------------------------- per-mode solve (sweep)
__global__ void __launch_bounds__(256) solve_kernel(const SolveArgs a) {
  __shared__ double sL[32 * 33];
  __shared__ double sUp[32 * 32];
  __shared__ double sX[256];   // rows x R of the new factor block (row-major)
  __shared__ double sB[256];   // rhs M + F (row-major)
  __shared__ double sM[256];   // M (row-major), for <M, A>
  __shared__ double sdot[2][32];
  __shared__ int sfail;
  const int R = a.R, RR = R * R;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (a.status[0] != 0.0) return;  // an earlier mode already failed

  // total Gram of the previous mode from its per-CTA partials (fixed order)
  if (a.gprev != nullptr) {
    for (int e = tid; e < RR; e += blockDim.x) {
      double s = 0.0;
      for (int c = 0; c < a.nprev; ++c) s += a.gprev[(int64_t)c * RR + e];
      sUp[e] = s;
      if (blockIdx.x == 0) a.Ups[(int64_t)a.prev_mode * RR + e] = s;
    }
    __syncthreads();
  }
  // Gamma^(n) = *_{k != n} Upsilon^(k)   (eq:Gamma)
  for (int e = tid; e < RR; e += blockDim.x) {
    double gm = 1.0;
    for (int k = 0; k < a.N; ++k) {
      if (k == a.mode) continue;
      gm *= (a.gprev != nullptr && k == a.prev_mode) ? sUp[e] : a.Ups[(int64_t)k * RR + e];
    }
    sL[(e % R) * 33 + (e / R)] = gm;
  }
  if (tid == 0) sfail = 0;
  __syncthreads();
  if (warp == 0) {
    const bool ok = warp_cholesky(sL, R, lane);
    if (!ok && lane == 0) sfail = 1;
  }
  __syncthreads();
  if (sfail) {
    if (blockIdx.x == 0 && tid == 0) {
      a.status[0] = (double)CP_ENOTSPD;
      a.status[1] = (double)a.mode;
    }
    return;
  }

  const int64_t In = a.In;
  const int64_t i0 = (int64_t)blockIdx.x * a.rpc;
  const int nrows = (int)((In - i0) < a.rpc ? (In - i0) : a.rpc);
  // phase A: M rows from the stream partials (+F): thread per (row, r)
  for (int e = tid; e < nrows * R; e += blockDim.x) {
    const int ii = e / R, r = e - (e / R) * R;
    const int64_t i = i0 + ii;
    const double m = reduce_entry(a.rg, i, r);
    sM[e] = m;
    sB[e] = m + (a.F != nullptr ? a.F[i + In * r] : 0.0);
  }
  __syncthreads();
  // phase B: warp per row, lane r: forward L y = b, back L^T x = y
  for (int ii = warp; ii < nrows; ii += blockDim.x / 32) {
    double b = (lane < R) ? sB[ii * R + lane] : 0.0;
    for (int k = 0; k < R; ++k) {
      const double yk = __shfl_sync(0xffffffffu, b / sL[k * 33 + k], k);
      if (lane == k) b = yk;
      if (lane > k && lane < R) b -= sL[lane * 33 + k] * yk;
    }
    for (int k = R - 1; k >= 0; --k) {
      const double xk = __shfl_sync(0xffffffffu, b / sL[k * 33 + k], k);
      if (lane == k) b = xk;
      if (lane < k) b -= sL[k * 33 + lane] * xk;
    }
    const int64_t i = i0 + ii;
    double dm = 0.0, df = 0.0;
    if (lane < R) {
      a.A[i + In * lane] = b;
      a.At[i * (R + (R & 1)) + lane] = b;
      sX[ii * R + lane] = b;
      dm = sM[ii * R + lane] * b;
      df = (a.F != nullptr) ? a.F[i + In * lane] * b : 0.0;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      dm += __shfl_xor_sync(0xffffffffu, dm, off);
      df += __shfl_xor_sync(0xffffffffu, df, off);
    }
    if (lane == 0) {
      sB[ii * R] = dm;  // reuse: row dots (rhs no longer needed for this row)
      sM[ii * R] = df;
    }
  }
  __syncthreads();
  // partial Gram of the new rows, and the CTA's <M,A>, <F,A> (fixed order)
  for (int e = tid; e < RR; e += blockDim.x) {
    const int r = e % R, s = e / R;
    double g = 0.0;
    for (int ii = 0; ii < nrows; ++ii) g = fma(sX[ii * R + r], sX[ii * R + s], g);
    a.gcur[(int64_t)blockIdx.x * RR + e] = g;
  }
  if (tid == 0) {
    double dm = 0.0, df = 0.0;
    for (int ii = 0; ii < nrows; ++ii) {
      dm += sB[ii * R];
      df += sM[ii * R];
    }
    a.dotM[blockIdx.x] = dm;
    a.dotF[blockIdx.x] = df;
  }
}

// ---------------------------------------------------------------- sweep finalize: f, f_tilde
__global__ void finalize_sweep_kernel(const FinalizeArgs a) {
  __shared__ double sUp[32 * 32];
  __shared__ double sred[256];
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
  for (int e = tid; e < RR; e += blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < a.nlast; ++c) s += a.glast[(int64_t)c * RR + e];
    sUp[e] = s;
    a.Ups[(int64_t)(a.N - 1) * RR + e] = s;
  }
  __syncthreads();
  // ||[[A]]||^2 = 1^T (*_k Upsilon^(k)) 1
  double m2 = 0.0;
  for (int e = tid; e < RR; e += blockDim.x) {
    double p = sUp[e];
    for (int k = 0; k < a.N - 1; ++k) p *= a.Ups[(int64_t)k * RR + e];
    m2 += p;
  }
  sred[tid] = m2;
  __syncthreads();
  if (tid == 0) {
    double model2 = 0.0;
    for (int t = 0; t < blockDim.x; ++t) model2 += sred[t];
    double inner = 0.0;
    for (int c = 0; c < a.nlast; ++c) inner += a.dotM_last[c];
    double fa = 0.0;
    for (int n = 0; n < a.N; ++n)
      for (int c = 0; c < a.nsolve[n]; ++c) fa += a.dotF[(int64_t)n * a.dot_stride + c];
    const double f = 0.5 * a.normZ2[0] - inner + 0.5 * model2;
    a.out[0] = f;
    a.out[1] = f - fa;
    a.out[2] = 0.0;
    a.out[3] = -1.0;
  }
}

// ---------------------------------------------------------------- gradient (cp_fit)
// G^(n)(i,r) = -M(i,r) + sum_s A(i,s) Gamma(s,r) - F(i,r)   (eq:gradEqn; FAS residual with F)
__global__ void __launch_bounds__(256) gradient_kernel(const GradArgs a) {
  __shared__ double sG[32 * 32];
  __shared__ double sred[256];
  const int R = a.R, RR = R * R, tid = threadIdx.x;
  for (int e = tid; e < RR; e += blockDim.x) {
    double gm = 1.0;
    for (int k = 0; k < a.N; ++k)
      if (k != a.mode) gm *= a.Ups[(int64_t)k * RR + e];
    sG[e] = gm;
  }
  __syncthreads();
  const int64_t In = a.In;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + tid;
  double g2 = 0.0;
  if (idx < In * R) {
    const int64_t i = idx % In;
    const int r = (int)(idx / In);
    double gv = -reduce_entry(a.rg, i, r);
    for (int s = 0; s < R; ++s) gv = fma(a.A[i + In * s], sG[s + R * r], gv);
    if (a.F != nullptr) gv -= a.F[idx];
    if (a.G != nullptr) a.G[idx] = gv;
    g2 = gv * gv;
  }
  sred[tid] = g2;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (tid < off) sred[tid] += sred[tid + off];
    __syncthreads();
  }
  if (tid == 0) a.gpart[blockIdx.x] = sred[0];
}

__global__ void finalize_fit_kernel(const FitFinalArgs a) {
  if (threadIdx.x != 0) return;
  double res = 0.0;
  for (int c = 0; c < a.nresid; ++c) res += a.resid[c];
  double tot = 0.0;
  for (int n = 0; n < a.N; ++n) {
    double s = 0.0;
    for (int c = 0; c < a.ngrad[n]; ++c) s += a.gpart[(int64_t)n * a.gstride + c];
    a.out[2 + n] = s;
    tot += s;
  }
  a.out[0] = 0.5 * res;
  a.out[1] = sqrt(tot) / sqrt(a.normZ2[0]);
}

// ---------------------------------------------------------------- ||Z||^2
__global__ void __launch_bounds__(512) norm2_kernel(const double *__restrict__ Z, int64_t P,
                                                    double *part) {
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

__global__ void norm2_final_kernel(const double *part, int n, double *out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int c = 0; c < n; ++c) s += part[c];
    out[0] = s;
  }
}

}  // namespace cpk
