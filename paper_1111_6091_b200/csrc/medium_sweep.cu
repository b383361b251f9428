// Fused ALS / BNGS sweeps for medium tensors (16384 < P <= kMediumSweepMaxP: c1 50^3, c2 100^3,
// the finest levels of their multigrid hierarchies) -- EXPERIMENTAL, opt-in (CP_MEDIUM_SWEEP=1):
// measured slower than the general multi-kernel path (DESIGN 6.7), kept parity-tested.
// ONE cooperative launch of G CTAs runs `nsweeps` complete sweeps (eq:gradEqn, eq:Gamma,
// eq:relaxinnersolve) with two grid barriers per mode:
//   phase A (CTA c): the columns q in [Q c / G, Q (c + 1) / G) of Z viewed as I_n x Q are staged
//     into shared memory with their Khatri-Rao weights w(q, r) (P:110 order), a warp per output
//     entry forms the partial M_c(i, r) (lanes stride q, fixed xor tree) -> global
//   barrier; CTA c sums the entries o = c (mod G) over all partials (fixed order) -> global M;
//   barrier; every CTA reads M
//   phase B (every CTA, redundantly and identically): + F; Gamma from the Grams; Cholesky (rsqrt
//     pivots); every row solved; the new Gram.  All CTAs hold bitwise-identical factor copies in
//     shared memory, so no broadcast is needed.
// f, f~ as cp_als_sweep (readings R5, R6), written by CTA 0.
#include <cstdlib>

#include "cp_internal.cuh"
#include "small_sweep.cuh"

namespace cpk {

namespace {
constexpr int kT = kSmallSweepThreads;

__device__ __forceinline__ double ms_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx, y * y, 1.5);
  y = y * fma(-hx, y * y, 1.5);
  return y;
}

__device__ double block_sum_fixed_m(double v, double *red) {
  const int tid = threadIdx.x;
  __syncthreads();
  red[tid] = v;
  __syncthreads();
  for (int off = kT / 2; off > 0; off >>= 1) {
    if (tid < off) red[tid] += red[tid + off];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

// grid barrier k (1-based) over G co-resident CTAs: arrive on a counter zeroed before the launch,
// spin until G k arrivals.  A spin bound turns a (never expected) hang into a reported failure.
__device__ bool grid_barrier(unsigned *cnt, unsigned target) {
  __syncthreads();
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(cnt, 1u);
    int ok = 1;
    unsigned v;
    long long spins = 0;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
      if (v >= target) break;
      if (++spins > (1ll << 26)) {
        ok = 0;
        break;
      }
      __nanosleep(spins < 8 ? 64 : 256);
    }
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}
}  // namespace

__global__ void __launch_bounds__(kSmallSweepThreads) medium_sweep_kernel(const SmallSweepArgs a) {
  griddep();
  extern __shared__ double sm[];
  const int tid = threadIdx.x, N = a.N, R = a.R, RR = R * R;
  const int G = gridDim.x, c = blockIdx.x;
  const int64_t P = a.P;
  __shared__ int s_aoff[CP_MAX_N], s_dims[CP_MAX_N];
  __shared__ int s_status, s_failed;
  __shared__ double sDi[kSmallSweepMaxR];
  // shared layout (doubles): A^(0..N-1) | Ups | M | y | W (slab weights) | Gam | L | red | Zs (slab)
  int64_t off = 0;
  for (int k = 0; k < N; ++k) {
    if (tid == 0) {
      s_aoff[k] = (int)off;
      s_dims[k] = (int)a.dims[k];
    }
    off += a.dims[k] * R;
  }
  double *sU = sm + off;
  off += (int64_t)N * RR;
  double *sM = sm + off;
  off += a.imax * R;
  double *sY = sm + off;
  off += a.imax * R;
  double *sW = sm + off;
  off += a.npart * R;  // npart: max columns per CTA over the modes
  double *sG = sm + off;
  off += RR;
  double *sL = sm + off;
  off += RR;
  double *red = sm + off;
  off += kT;
  double *sZs = sm + off;  // slab: I_n x nq (column-major, column stride I_n)
  __syncthreads();
  for (int k = 0; k < N; ++k)
    for (int e = tid; e < s_dims[k] * R; e += kT) (sm + s_aoff[k])[e] = a.A[k][e];
  if (tid == 0) {
    s_status = 0;
    s_failed = -1;
  }
  __syncthreads();
  for (int e = tid; e < N * RR; e += kT) {
    const int k = e / RR, rs = e - k * RR, r = rs % R, s = rs / R;
    const double *x = (sm + s_aoff[k]) + s_dims[k] * r, *y = (sm + s_aoff[k]) + s_dims[k] * s;
    double g = 0.0;
    for (int i = 0; i < s_dims[k]; ++i) g = fma(x[i], y[i], g);
    sU[e] = g;
  }
  __syncthreads();

  unsigned nbar = 0;
  double inner_last = 0.0;
  for (int sweep = 0; sweep < a.nsweeps && s_status == 0; ++sweep) {
    for (int n = 0; n < N; ++n) {
      const int In = s_dims[n];
      int left = 1;
      for (int k = 0; k < n; ++k) left *= s_dims[k];
      const int Q = (int)(P / In);
      const int q0 = (int)(((int64_t)Q * c) / G), q1 = (int)(((int64_t)Q * (c + 1)) / G);
      const int nq = q1 - q0;
      // ---- phase A: stage the slab and its Khatri-Rao weights (32-bit index math) ----
      {
        // walk (i fastest, then q) with an incremental (aa, b) odometer per thread stride
        for (int e = tid; e < In * nq; e += kT) {
          const int qq = e / In, i = e - qq * In;
          const int q = q0 + qq, b = q / left, aa = q - b * left;
          sZs[e] = __ldg(a.Z + (aa + left * (i + In * b)));
        }
      }
      for (int e = tid; e < nq * R; e += kT) {
        const int qq = e % nq, r = e / nq;
        int q = q0 + qq;
        double w = 1.0;
        for (int k = 0; k < N; ++k) {  // q = Kolda-order index over the modes k != n
          if (k == n) continue;
          const int Ik = s_dims[k];
          const int ik = q % Ik;
          q /= Ik;
          w *= (sm + s_aoff[k])[ik + Ik * r];
        }
        sW[qq + nq * r] = w;
      }
      __syncthreads();
      const int nout = In * R;
      double *part = a.mpart + (int64_t)((nbar >> 1) & 1) * G * a.imax * R;
      {
        const int warp = tid >> 5, lane = tid & 31;
        for (int o = warp; o < nout; o += kT / 32) {
          const int i = o % In, r = o / In;
          const double *w = sW + nq * r;
          double acc = 0.0;
          for (int qq = lane; qq < nq; qq += 32) acc = fma(sZs[i + (int64_t)In * qq], w[qq], acc);
#pragma unroll
          for (int o2 = 16; o2 > 0; o2 >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o2);
          if (lane == 0) part[(int64_t)c * nout + o] = acc;
        }
      }
      ++nbar;
      if (!grid_barrier(a.bar, nbar * (unsigned)G)) {
        if (tid == 0) {
          s_status = CP_ECUDA;
          s_failed = n;
        }
        __syncthreads();
        break;
      }
      // ---- the partial sums: CTA c reduces the entries o = c (mod G) over all CTAs (c order),
      // a second barrier, then every CTA reads the whole M ----
      {
        double *mfull = a.mpart + (int64_t)2 * G * a.imax * R;
        const int warp = tid >> 5, lane = tid & 31;
        for (int o = c + G * warp; o < nout; o += G * (kT / 32)) {
          double m = 0.0;
          for (int cc = lane; cc < G; cc += 32) m += __ldcg(part + (int64_t)cc * nout + o);
#pragma unroll
          for (int o2 = 16; o2 > 0; o2 >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o2);
          if (lane == 0) mfull[o] = m;
        }
        ++nbar;
        if (!grid_barrier(a.bar, nbar * (unsigned)G)) {
          if (tid == 0) {
            s_status = CP_ECUDA;
            s_failed = n;
          }
          __syncthreads();
          break;
        }
        for (int o = tid; o < nout; o += kT) sM[o] = __ldcg(mfull + o);
      }
      // ---- phase B (identical in every CTA) ----
      for (int e = tid; e < RR; e += kT) {
        double g = 1.0;
        for (int k = 0; k < N; ++k)
          if (k != n) g *= sU[k * RR + e];
        sG[e] = g;
      }
      __syncthreads();
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
          const double rj = ms_rsqrt(d), ljj = d * rj;
          sL[j + R * j] = ljj;
          sDi[j] = rj;
          for (int i = j + 1; i < R; ++i) {
            double s = sG[i + R * j];
            for (int k = 0; k < j; ++k) s -= sL[i + R * k] * sL[j + R * k];
            sL[i + R * j] = s * rj;
          }
        }
      }
      __syncthreads();
      if (s_status != 0) break;
      const double *F = a.F[n];
      double *An = sm + s_aoff[n];
      for (int i = tid; i < In; i += kT) {
        double *y = sY + (int64_t)i * R;
        for (int r = 0; r < R; ++r) {
          double b = sM[i + In * r] + (F != nullptr ? F[i + In * r] : 0.0);
          for (int k = 0; k < r; ++k) b -= sL[r + R * k] * y[k];
          y[r] = b * sDi[r];
        }
        for (int r = R - 1; r >= 0; --r) {
          double x = y[r];
          for (int k = r + 1; k < R; ++k) x -= sL[k + R * r] * y[k];
          y[r] = x * sDi[r];
          An[i + In * r] = y[r];
        }
      }
      __syncthreads();
      for (int e = tid; e < RR; e += kT) {
        const int r = e % R, s = e / R;
        const double *x = An + In * r, *y = An + In * s;
        double g = 0.0;
        for (int i = 0; i < In; ++i) g = fma(x[i], y[i], g);
        sU[n * RR + e] = g;
      }
      if (n == N - 1 && sweep == a.nsweeps - 1) {
        double d = 0.0;
        for (int o = tid; o < nout; o += kT) d = fma(sM[o], An[o], d);
        inner_last = block_sum_fixed_m(d, red);
      }
      __syncthreads();
    }
  }
  if (c != 0) return;
  // ---- CTA 0: write back, f and f~ (readings R6, R5) ----
  for (int k = 0; k < N; ++k)
    for (int e = tid; e < s_dims[k] * R; e += kT) a.A[k][e] = (sm + s_aoff[k])[e];
  if (s_status != 0) {
    if (tid == 0) {
      a.out[0] = nan("");
      a.out[1] = nan("");
      a.out[2] = (double)s_status;
      a.out[3] = (double)s_failed;
    }
    return;
  }
  double m2 = 0.0;
  for (int e = tid; e < RR; e += kT) {
    double p = 1.0;
    for (int k = 0; k < N; ++k) p *= sU[k * RR + e];
    m2 += p;
  }
  const double model2 = block_sum_fixed_m(m2, red);
  double fa = 0.0;
  for (int k = 0; k < N; ++k)
    if (a.F[k] != nullptr)
      for (int e = tid; e < s_dims[k] * R; e += kT) fa = fma(a.F[k][e], (sm + s_aoff[k])[e], fa);
  const double fas = block_sum_fixed_m(fa, red);
  if (tid == 0) {
    const double f = 0.5 * a.normZ2[0] - inner_last + 0.5 * model2;
    a.out[0] = f;
    a.out[1] = f - fas;
    a.out[2] = 0.0;
    a.out[3] = -1.0;
  }
}

// CTAs of the medium kernel for shape s (0: not applicable).  About 6 K tensor elements per
// CTA, at most one CTA per SM (co-residency of the grid barrier is guaranteed by the
// cooperative launch).
int medium_sweep_ctas(const cp_shape &s, int sms) {
  if (s.R > kSmallSweepMaxR) return 0;
  double P = 1.0;
  for (int k = 0; k < s.N; ++k) P *= (double)s.dims[k];
  if (P <= (double)kSmallSweepMaxP || P > (double)kMediumSweepMaxP) return 0;
  static const double per = [] {
    const char *e = getenv("CP_MEDIUM_ELEMS");
    return (e && *e) ? atof(e) : 6144.0;
  }();
  int G = (int)((P + per - 1.0) / per);
  if (G > sms) G = sms;
  if (G < 2) G = 2;
  return G;
}

size_t medium_sweep_smem_bytes(const cp_shape &s, int G) {
  double P = 1.0;
  int64_t imax = 1, sumI = 0, minI = s.dims[0];
  for (int k = 0; k < s.N; ++k) {
    P *= (double)s.dims[k];
    sumI += s.dims[k];
    if (s.dims[k] > imax) imax = s.dims[k];
    if (s.dims[k] < minI) minI = s.dims[k];
  }
  const double nqmax = P / (double)minI / G + 1.0;  // max columns per CTA over the modes
  const double slab = P / G + (double)imax + 1.0;   // >= I_n * nq for every mode
  const double d = (double)sumI * s.R + (double)s.N * s.R * s.R + 2.0 * imax * s.R + nqmax * s.R +
                   2.0 * s.R * s.R + kT + slab + 8.0;
  return (size_t)(d * 8.0);
}

size_t medium_sweep_ws_doubles(const cp_shape &s, int G) {
  int64_t imax = 1;
  for (int k = 0; k < s.N; ++k)
    if (s.dims[k] > imax) imax = s.dims[k];
  return (size_t)(2 * (int64_t)G * imax * s.R + imax * s.R + 32);  // 2 partial buffers + M
}

cudaError_t launch_medium_sweep(const cp_shape &s, int G, const double *Z, const double *normZ2, double *const *A,
                                const double *const *F, int nsweeps, double *out, double *ws, cudaStream_t st) {
  SmallSweepArgs a;
  memset(&a, 0, sizeof(a));
  a.N = s.N;
  a.R = s.R;
  a.nsweeps = nsweeps;
  a.P = 1;
  a.imax = 1;
  int64_t minI = s.dims[0];
  for (int k = 0; k < s.N; ++k) {
    a.dims[k] = s.dims[k];
    a.P *= s.dims[k];
    if (s.dims[k] > a.imax) a.imax = s.dims[k];
    if (s.dims[k] < minI) minI = s.dims[k];
    a.A[k] = A[k];
    a.F[k] = (F != nullptr) ? F[k] : nullptr;
  }
  a.npart = a.P / minI / G + 1;
  a.Z = Z;
  a.normZ2 = normZ2;
  a.out = out;
  a.bar = reinterpret_cast<unsigned *>(ws);
  a.mpart = ws + 32;
  const size_t smem = medium_sweep_smem_bytes(s, G);
  static size_t attr_set = 0;
  if (smem > 48 * 1024 && smem > attr_set) {
    cudaError_t e = cudaFuncSetAttribute(medium_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = smem;
  }
  cudaError_t e = cudaMemsetAsync(a.bar, 0, 8, st);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, medium_sweep_kernel, a);
}

}  // namespace cpk
