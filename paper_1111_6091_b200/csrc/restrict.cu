// restrict.cu -- cp_restrict_structured: X = Z x_n Phat^T for the transfer operator of the
// geometric C/F splitting.
//
// P (I x Ic) injects the C points (P(2j, j) = 1) and interpolates each F point 2j+1 from its
// coarse neighbours j, j+1 with the weights wl, wr of the least-squares fit.  B = P^T P is then
// tridiagonal,
//     B(j, j)   = 1 + wr[2j-1]^2 + wl[2j+1]^2,     B(j, j-1) = wl[2j-1] wr[2j-1],
// so its Cholesky factor L is lower bidiagonal (diagonal ld, sub-diagonal le) and
//     Phat = P L^{-T},  Phat^T = L^{-1} P^T:
//     y_j = z_{2j} + wr[2j-1] z_{2j-1} + wl[2j+1] z_{2j+1}      (P^T along the fiber: 3 taps)
//     x_j = (y_j - le_j x_{j-1}) / ld_j                         (L x = y: forward substitution)
// for every fiber of mode n.  One pass over Z (8P bytes read, 8P Ic/I written), O(P) flops:
// HBM-bound, where the dense product costs 2 Ic P flops (fp64-bound).  Derived here (SURVEY
// NEXT-3), not in the paper, which costs the Galerkin tensor as O(PS).
//
// Kernels: restrict_factor_kernel (one warp: B and its bidiagonal factor, a coefficient table
// coef[j] = {cA_j = wr[2j-1], cB_j = wl[2j+1], le_j, 1/ld_j}); restrict_tma_kernel (mode n >= 1,
// default: 1-KB row slabs of 128 fibers streamed by bulk copies through an mbarrier ring);
// restrict_inner_kernel (mode n >= 1 fallback: thread per fiber, coalesced loads);
// restrict_mode0_kernel (mode 0: fibers are contiguous rows; 128-fiber tiles are staged
// through shared memory so both the loads and the stores are coalesced).
#include <cstdlib>

#include "cp_internal.cuh"

namespace cpk {

// one coefficient entry (32 bytes, LDG.256 through the read-only path)
__device__ __forceinline__ double4 coef_at(const double *coef, int64_t j) {
  double4 c;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(c.x), "=d"(c.y), "=d"(c.z), "=d"(c.w) : "l"(coef + 4 * j));
  return c;
}

// coefficient table (4 doubles per coarse point) from the weights; lanes form B's entries,
// lane 0 runs the O(Ic) factor recurrence (the only sequential step)
__global__ void __launch_bounds__(32) restrict_factor_kernel(const double *wl, const double *wr, int64_t I,
                                                            int64_t Ic, double *coef) {
  griddep();
  for (int64_t j = threadIdx.x; j < Ic; j += 32) {
    const double cA = (j >= 1) ? wr[2 * j - 1] : 0.0;
    const double cB = (2 * j + 1 < I) ? wl[2 * j + 1] : 0.0;
    const double sub = (j >= 1) ? wl[2 * j - 1] * wr[2 * j - 1] : 0.0;  // B(j, j-1)
    coef[4 * j + 0] = cA;
    coef[4 * j + 1] = cB;
    coef[4 * j + 2] = sub;                                   // le_j after the recurrence
    coef[4 * j + 3] = fma(cA, cA, fma(cB, cB, 1.0));          // B(j, j), then 1 / ld_j
  }
  __syncwarp();
  if (threadIdx.x == 0) {
    // le_j = B(j, j-1) / ld_{j-1},  ld_j = sqrt(B(j, j) - le_j^2); carried as 1 / ld (an
    // rsqrt refined by two Newton steps: no division or square root on the serial chain)
    double inv_prev = 0.0;
    for (int64_t j = 0; j < Ic; ++j) {
      const double le = coef[4 * j + 2] * inv_prev;
      const double q = fma(-le, le, coef[4 * j + 3]);
      double y;
      asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
      const double hq = 0.5 * q;
      y = y * fma(-hq, y * y, 1.5);
      y = y * fma(-hq, y * y, 1.5);
      coef[4 * j + 2] = le;
      coef[4 * j + 3] = y;
      inv_prev = y;
    }
  }
}

// mode n >= 1: fiber (o, s) = elements o * I * S + i * S + s, i < I.  V consecutive fibers per
// thread (V = 2: 16-byte loads and stores, 512-byte warp requests; needs S even and 16-byte
// aligned tensors)
template <int V>
struct vec_t;
template <>
struct vec_t<1> {
  using T = double;
  static __device__ __forceinline__ double get(const T &v, int) { return v; }
  static __device__ __forceinline__ void set(T &v, int, double x) { v = x; }
};
template <>
struct vec_t<2> {
  using T = double2;
  static __device__ __forceinline__ double get(const T &v, int u) { return u ? v.y : v.x; }
  static __device__ __forceinline__ void set(T &v, int u, double x) {
    if (u) v.y = x;
    else v.x = x;
  }
};

template <int V>
__global__ void __launch_bounds__(256) restrict_inner_kernel(const double *__restrict__ Z, int64_t I, int64_t Ic,
                                                             int64_t S, int64_t nfib, const double *__restrict__ coef,
                                                             double *__restrict__ X) {
  using VT = typename vec_t<V>::T;
  griddep();  // (every read of Z after the wait: Z may be the output of an earlier kernel)
  const int64_t f = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * V;  // first fiber of the thread
  const int64_t o = f / S, s = f - (f / S) * S;
  const VT *z = reinterpret_cast<const VT *>(Z + o * I * S + s);
  VT *x = reinterpret_cast<VT *>(X + o * Ic * S + s);
  const int64_t Sv = S / V;  // stride in vectors
  VT zprev, xprev, z0, z1;
#pragma unroll
  for (int u = 0; u < V; ++u) {
    vec_t<V>::set(zprev, u, 0.0);
    vec_t<V>::set(xprev, u, 0.0);
    vec_t<V>::set(z1, u, 0.0);
  }
  if (f >= nfib) return;
  z0 = __ldcs(z);
  if (I > 1) z1 = __ldcs(z + Sv);
  auto step = [&](const double4 &c, const VT &zc, const VT &zf, int64_t j) {
    VT xv;
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const double y = fma(c.y, vec_t<V>::get(zf, u), fma(c.x, vec_t<V>::get(zprev, u), vec_t<V>::get(zc, u)));
      vec_t<V>::set(xv, u, fma(-c.z, vec_t<V>::get(xprev, u), y) * c.w);
    }
    __stcs(x + j * Sv, xv);
    zprev = zf;
    xprev = xv;
  };
  step(coef_at(coef, 0), z0, z1, 0);
  int64_t j = 1;
  // 4 coarse points per iteration: the 8 loads of Z are issued before the recurrence
  for (; 2 * (j + 3) + 1 < I; j += 4) {
    VT zc[4], zf[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      zc[u] = __ldcs(z + (2 * (j + u)) * Sv);
      zf[u] = __ldcs(z + (2 * (j + u) + 1) * Sv);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) step(coef_at(coef, j + u), zc[u], zf[u], j + u);
  }
  for (; j < Ic; ++j) {
    const VT zc = __ldcs(z + (2 * j) * Sv);
    VT zf = zc;
    if (2 * j + 1 < I) zf = __ldcs(z + (2 * j + 1) * Sv);
    else
#pragma unroll
      for (int u = 0; u < V; ++u) vec_t<V>::set(zf, u, 0.0);
    step(coef_at(coef, j), zc, zf, j);
  }
}

// mode n >= 1, TMA version: a block owns a slab of kRtW consecutive inner indices s (one fiber
// per thread) of one outer index o and streams its I rows (kRtW doubles = 1 KB each, contiguous)
// through a ring of kRtNS shared-memory stages of kRtRows rows, one bulk copy per row
// (cp.async.bulk + mbarrier transaction counts).  Big contiguous requests, deep pipelining;
// the recurrence reads the stage from shared memory.  Needs S even (16-byte rows).
constexpr int kRtW = 128, kRtRows = 8, kRtNS = 5;  // 40 KB of stages: ~5 blocks per SM
__global__ void __launch_bounds__(kRtW) restrict_tma_kernel(const double *__restrict__ Z, int64_t I, int64_t Ic,
                                                           int64_t S, int64_t nslab,
                                                           const double *__restrict__ coef, double *__restrict__ X) {
  griddep();
  __shared__ __align__(128) double tz[kRtNS][kRtRows][kRtW];
  __shared__ __align__(8) uint64_t full[kRtNS];
  const int t = threadIdx.x;
  const int64_t o = blockIdx.x / nslab, sb = (blockIdx.x % nslab) * kRtW;
  const int w = (int)((S - sb) < kRtW ? (S - sb) : kRtW);  // slab width (even)
  const double *zb = Z + o * I * S + sb;
  double *xb = X + o * Ic * S + sb;
  const int nst = (int)((I + kRtRows - 1) / kRtRows);
  if (t == 0) {
    for (int q = 0; q < kRtNS; ++q) mbar_init(&full[q], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int st) {  // thread 0: rows st * kRtRows .. of the slab into slot st % kRtNS
    const int slot = st % kRtNS;
    const int64_t r0 = (int64_t)st * kRtRows;
    const int nr = (int)((I - r0) < kRtRows ? (I - r0) : kRtRows);
    mbar_expect_tx(&full[slot], (uint32_t)(nr * w * 8));
    for (int r = 0; r < nr; ++r) bulk_g2s(&tz[slot][r][0], zb + (r0 + r) * S, (uint32_t)(w * 8), &full[slot]);
    mbar_arrive(&full[slot]);  // the phase completes with this arrival and the landed bytes
  };
  if (t == 0)
    for (int st = 0; st < kRtNS && st < nst; ++st) issue(st);
  double zprev = 0.0, xprev = 0.0;
  for (int st = 0; st < nst; ++st) {
    const int slot = st % kRtNS;
    mbar_wait(&full[slot], (uint32_t)((st / kRtNS) & 1));
    const int64_t r0 = (int64_t)st * kRtRows;  // even: the stage starts at a C point
    const int nr = (int)((I - r0) < kRtRows ? (I - r0) : kRtRows);
    if (t < w) {
      for (int q = 0; q < nr; q += 2) {
        const int64_t j = (r0 + q) / 2;
        const double4 c = coef_at(coef, j);
        const double zc = tz[slot][q][t];
        const double zf = (q + 1 < nr) ? tz[slot][q + 1][t] : 0.0;
        const double y = fma(c.y, zf, fma(c.x, zprev, zc));
        const double xv = fma(-c.z, xprev, y) * c.w;
        __stcs(xb + j * S + t, xv);
        zprev = zf;
        xprev = xv;
      }
    }
    __syncthreads();  // every thread is done with the slot
    if (t == 0 && st + kRtNS < nst) issue(st + kRtNS);
  }
}

// mode 0: fibers are the contiguous rows of Z (length I); a block stages 128 rows x 32 fine
// columns (one chunk) in shared memory, each thread runs its row's recurrence over the chunk's
// 16 coarse points, and the 128 x 16 outputs leave through the same tile
constexpr int kR0Rows = 128, kR0Chunk = 32;
__global__ void __launch_bounds__(kR0Rows) restrict_mode0_kernel(const double *__restrict__ Z, int64_t I, int64_t Ic,
                                                                 int64_t nfib, const double *__restrict__ coef,
                                                                 double *__restrict__ X) {
  griddep();  // (every read of Z after the wait: Z may be the output of an earlier kernel)
  __shared__ double tz[kR0Rows][kR0Chunk + 1];  // the chunk; outputs overwrite it in place
                                                 // (x_jj lands in column jj <= 2 jj, already read)
  const int t = threadIdx.x;
  const int64_t f0 = (int64_t)blockIdx.x * kR0Rows;
  const int nrow = (int)((nfib - f0) < kR0Rows ? (nfib - f0) : kR0Rows);
  // software pipeline: the next chunk's 32 values per thread are loaded into registers while
  // the current chunk is solved and stored (consecutive threads read consecutive columns)
  double nxt[kR0Chunk];
  auto load_chunk = [&](int64_t c0) {
    const int ncol = (int)((I - c0) < kR0Chunk ? (I - c0) : kR0Chunk);
#pragma unroll
    for (int q = 0; q < kR0Chunk; ++q) {
      const int idx = q * kR0Rows + t;
      const int r = idx / kR0Chunk, k = idx % kR0Chunk;
      nxt[q] = (r < nrow && k < ncol) ? __ldcs(Z + (f0 + r) * I + c0 + k) : 0.0;
    }
  };
  load_chunk(0);
  double zprev = 0.0, xprev = 0.0;
  for (int64_t c0 = 0; c0 < I; c0 += kR0Chunk) {
#pragma unroll
    for (int q = 0; q < kR0Chunk; ++q) {
      const int idx = q * kR0Rows + t;
      tz[idx / kR0Chunk][idx % kR0Chunk] = nxt[q];
    }
    __syncthreads();
    if (c0 + kR0Chunk < I) load_chunk(c0 + kR0Chunk);
    const int64_t j0 = c0 / 2;
    const int nj = (int)((Ic - j0) < kR0Chunk / 2 ? (Ic - j0) : kR0Chunk / 2);
    for (int jj = 0; jj < nj; ++jj) {
      const double4 c = coef_at(coef, j0 + jj);
      const double zc = tz[t][2 * jj];
      const double zf = tz[t][2 * jj + 1];  // 0 beyond the last column (one-sided right end)
      const double y = fma(c.y, zf, fma(c.x, zprev, zc));
      const double xv = fma(-c.z, xprev, y) * c.w;
      tz[t][jj] = xv;
      zprev = zf;
      xprev = xv;
    }
    __syncthreads();
#pragma unroll 4
    for (int q = 0; q < kR0Chunk / 2; ++q) {
      const int idx = q * kR0Rows + t;
      const int r = idx / (kR0Chunk / 2), k = idx % (kR0Chunk / 2);
      if (r < nrow && k < nj) __stcs(X + (f0 + r) * Ic + j0 + k, tz[r][k]);
    }
    __syncthreads();
  }
}

}  // namespace cpk

using namespace cpk;

static size_t restrict_ws_doubles(int64_t I) { return (size_t)4 * ((I + 1) / 2); }

extern "C" size_t cp_restrict_workspace_bytes(int32_t N, const int64_t *dims, int32_t mode) {
  if (N < 1 || N > CP_MAX_N || dims == nullptr || mode < 0 || mode >= N || dims[mode] < 1) return 0;
  return restrict_ws_doubles(dims[mode]) * sizeof(double);
}

extern "C" int cp_restrict_structured(int32_t N, const int64_t *dims, const double *Z, int32_t mode,
                                      const double *wl, const double *wr, double *X, void *ws, size_t ws_bytes,
                                      cp_stream_t stream) {
  if (N < 1 || N > CP_MAX_N || dims == nullptr || mode < 0 || mode >= N) return CP_EINVAL;
  if (Z == nullptr || wl == nullptr || wr == nullptr || X == nullptr || ws == nullptr) return CP_EINVAL;
  double P = 1.0;
  for (int k = 0; k < N; ++k) {
    if (dims[k] < 1) return CP_EDIM;
    P *= (double)dims[k];
  }
  if (P >= 4611686018427387904.0) return CP_EDIM;
  const int64_t I = dims[mode], Ic = (I + 1) / 2;
  if (ws_bytes < restrict_ws_doubles(I) * sizeof(double) || ((uintptr_t)ws % 32) != 0) return CP_EWORKSPACE;
  int64_t S = 1, O = 1;
  for (int k = 0; k < mode; ++k) S *= dims[k];
  for (int k = mode + 1; k < N; ++k) O *= dims[k];
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  double *coef = static_cast<double *>(ws);
  if (launch_k(restrict_factor_kernel, dim3(1), dim3(32), 0, st, wl, wr, I, Ic, coef) != cudaSuccess)
    return CP_ECUDA;
  cudaError_t e;
  if (mode == 0) {
    const int64_t nfib = O;
    e = launch_k(restrict_mode0_kernel, dim3((unsigned)((nfib + kR0Rows - 1) / kR0Rows)), dim3(kR0Rows), 0, st, Z, I,
                 Ic, nfib, (const double *)coef, X);
  } else {
    const int64_t nfib = S * O;
    const bool v2 = (S % 2 == 0) && ((uintptr_t)Z % 16 == 0) && ((uintptr_t)X % 16 == 0);
    const int64_t nthr = v2 ? nfib / 2 : nfib;
    const int bs = knob("CP_RESTRICT_BLOCK", 128);  // 128: ~7 blocks per SM, small tail
    const bool tma = knob("CP_RESTRICT_TMA", 1) != 0 && (S % 2 == 0) && ((uintptr_t)Z % 16 == 0);
    if (tma) {
      const int64_t nslab = (S + kRtW - 1) / kRtW;
      e = launch_k(restrict_tma_kernel, dim3((unsigned)(O * nslab)), dim3(kRtW), 0, st, Z, I, Ic, S, nslab,
                   (const double *)coef, X);
    } else if (v2)
      e = launch_k(restrict_inner_kernel<2>, dim3((unsigned)((nthr + bs - 1) / bs)), dim3(bs), 0, st, Z, I, Ic, S, nfib,
                   (const double *)coef, X);
    else
      e = launch_k(restrict_inner_kernel<1>, dim3((unsigned)((nthr + bs - 1) / bs)), dim3(bs), 0, st, Z, I, Ic, S, nfib,
                   (const double *)coef, X);
  }
  return e == cudaSuccess ? CP_OK : CP_ECUDA;
}
