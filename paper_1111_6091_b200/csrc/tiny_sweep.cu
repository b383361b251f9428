// Two-warp ALS / BNGS sweeps for the tiniest tensors of the multigrid hierarchy (the coarsest
// levels: c1 and the paper's dense problems end at 4^3, where the V-cycle runs nu_c = 50
// relaxation sweeps, Table 1).
//
// The 512-thread fused kernel (small_sweep.cu) is latency-bound there: each of its ~8 phases per
// mode is a few hundred flops behind a 16-warp barrier (4^3, R = 3: 9.4 us per sweep).  Here one
// warp runs the data path of the whole call and a second one the R x R side beside it: Z, the
// factors, F and the Grams live in shared memory, phases are separated by __syncwarp and two
// 64-thread named barriers per mode, every lane factors the R x R Gamma redundantly in registers
// (no shuffles or pivot broadcasts on the chain), and a lane owns a row of the solve.  Same
// arithmetic definition and contract as small_sweep_kernel (for n = 1..N, M = Z_(n)Phi^(n)
// (eq:gradEqn), Gamma = *_{k != n} A^(k)T A^(k) (eq:Gamma), A^(n) Gamma = M + F
// (eq:relaxinnersolve P:356-358) by Cholesky without pivoting (reading R1); f, f~ of the last
// sweep by the expansion (readings R5, R6); optional eq:ALSnorm after every sweep), every sum
// in a fixed order (bitwise reproducible).
//
// The factor updates are BITWISE those of small_sweep_kernel: the same expressions in the same
// order everywhere, including the MTTKRP sums -- shapes are limited to modes with at most 32
// columns (left x right <= 32), where the fused kernel's "lanes stride the columns, xor tree" sum
// is one term per lane and a tree over the next power of two >= Q lanes (the upper lanes add
// exact zeros).  So switching kernels does not move a multigrid trajectory (the c1 solve is
// sensitive to rounding-level changes on its coarsest level: DESIGN reading R31).  Only f and f~
// (sums over lanes instead of threads) differ at rounding level.
#include "cp_internal.cuh"
#include "small_sweep.cuh"

#ifdef CP_TINY_TIMING
#include <cstdio>
#define TT(k) tt[k] = clock64();
#else
#define TT(k)
#endif

namespace cpk {

namespace {
constexpr int kTinyMaxN = 4;
constexpr int kTinyMaxA = 256;   // sum_k I_k R
constexpr int kTinyMaxW = 160;   // max_n (left + right) R
constexpr int kTinyMaxM = 128;   // max_n I_n R

__device__ __forceinline__ double ts_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx, y * y, 1.5);
  y = y * fma(-hx, y * y, 1.5);
  return y;
}

// x / d for 0 <= x < 2^22, d >= 1, from a float reciprocal plus one correction (exact)
__device__ __forceinline__ int ts_qdiv(int x, int d, float inv) {
  int q = __float2int_rz((float)x * inv);
  const int r = x - q * d;
  q += (r >= d) - (r < 0);
  return q;
}

// fixed xor tree over the warp; every lane gets the sum
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}
}  // namespace

// M(i, r) for the output entries o = i + In r: the PARTS = 2^ceil(log2 Q) column terms
// z(a, i, b) (WL(a, r) WR(b, r)) of an entry (columns q >= Q: 0) are summed in the order of
// small_sweep_kernel's 32-lane xor tree (level d: t[q] += t[q + d] for q < d, d = PARTS/2 .. 1;
// its levels above PARTS add exact zeros).  qt[q] = (a + bstride b, a, b) of column q (built
// once per call).
template <int PARTS>
__device__ __noinline__ void tiny_mttkrp(const double *sZ, const double *sWL, const double *sWR, double *sM,
                                         const ushort4 *qt, int Q, int left, int right, int In, float inv_In, int nout,
                                         int lane) {
  // Two lanes per output entry: lane parity h takes the columns q = 2 j + h and runs the tree's
  // levels PARTS/2 .. 2 in its registers (they only pair columns of equal parity); the last level,
  // t[0] + t[1], is one shuffle.  PARTS = 1: one lane, one term.
  constexpr int H = PARTS > 1 ? PARTS / 2 : 1;
  const int h = PARTS > 1 ? (lane & 1) : 0;
  const int per = PARTS > 1 ? 16 : 32;  // output entries per round
  for (int o0 = 0; o0 < nout; o0 += per) {
    const int o = o0 + (PARTS > 1 ? (lane >> 1) : lane);
    const int oc = o < nout ? o : 0;
    const int r = ts_qdiv(oc, In, inv_In), i = oc - r * In;
    const double *zrow = sZ + left * i, *wl = sWL + left * r, *wr = sWR + right * r;
    // branch-free (columns q >= Q re-read column 0 and are zeroed by a select): with a branch per
    // column the terms ran one after the other, ~110 cycles each
    double t[H];
    ushort4 cq[H];
#pragma unroll
    for (int j = 0; j < H; ++j) {
      const int q = (PARTS > 1 ? 2 * j : j) + h;
      cq[j] = qt[q < Q ? q : 0];
    }
#pragma unroll
    for (int j = 0; j < H; ++j) {
      const int q = (PARTS > 1 ? 2 * j : j) + h;
      const double v = fma(zrow[cq[j].x], wl[cq[j].y] * wr[cq[j].z], 0.0);
      t[j] = (q < Q) ? v : 0.0;
    }
#pragma unroll
    for (int d = H / 2; d > 0; d >>= 1)
#pragma unroll
      for (int j = 0; j < d; ++j) t[j] += t[j + d];
    double m = t[0];
    if (PARTS > 1) {
      const double other = __shfl_xor_sync(0xffffffffu, m, 1);
      m = m + other;  // (h = 0: t[0] + t[1], the tree's last level)
    }
    if (h == 0 && o < nout) sM[o] = m;
  }
}

// (The mode loops are unrolled with the per-mode sizes in registers.  A rolled variant with the
// sizes in shared memory -- one copy of the per-mode code -- measured slower: 4^3 R = 3 357 vs
// 272 us per 50 sweeps; the rolled Gamma product alone went from ~400 to ~2350 cycles per mode.)
template <int R>
__global__ void __launch_bounds__(64) tiny_sweep_kernel(const SmallSweepArgs a) {
  griddep();
  constexpr int RR = R * R;
  constexpr int MN = kTinyMaxN;
  // Two warps: warp 0 runs the data path of every mode (Khatri-Rao halves, MTTKRP, row solves),
  // warp 1 the R x R side (Upsilon of the factor just solved, Gamma of the next mode and its
  // Cholesky factor, handed over through shared memory) -- the same arithmetic as one warp doing
  // both in turn, with the factorization off the data path's chain.  Named barriers: kBarL (L of
  // the mode is ready / the solve may start), kBarA (the solved factor is ready for its Gram).
  constexpr int kBarL = 1, kBarA = 2, kBarS = 3;
  __shared__ double sL[R * R], sDi[R];
  __shared__ int s_status, s_failed;
  __shared__ double s_model2;
  const int warp = threadIdx.x >> 5;
  __shared__ double sZ[kTinySweepMaxP];
  __shared__ double sA[kTinyMaxA + 1], sF[kTinyMaxA];  // sA[kTinyMaxA] = 1.0
  __shared__ double sW[kTinyMaxW];
  __shared__ double sM[kTinyMaxM];
  __shared__ double sU[MN * RR];
  // Khatri-Rao half entry ee of mode n = product of up to 3 factor entries: their offsets in sA
  // (unused slots point at the 1.0), built once per call
  __shared__ ushort4 sTab[MN][kTinyMaxW];
  __shared__ ushort4 sQt[MN][32];  // column q of mode n: (a + bstride b, a, b)
  __shared__ double sNrm[MN * R], sLam[R];
  __shared__ int sPos[R];
  const int lane = threadIdx.x & 31, N = a.N, tid = threadIdx.x;
  const int P = (int)a.P;
  int dims[MN], aoff[MN];
  float invd[MN];
  int off = 0;
  bool anyF = false;
#pragma unroll
  for (int k = 0; k < MN; ++k) {
    dims[k] = (k < N) ? (int)a.dims[k] : 1;
    invd[k] = 1.0f / (float)dims[k];
    aoff[k] = off;
    if (k < N) off += dims[k] * R;
    if (k < N && a.F[k] != nullptr) anyF = true;
  }
  for (int e = tid; e < P; e += 64) sZ[e] = a.Z[e];
#pragma unroll
  for (int k = 0; k < MN; ++k) {
    if (k < N) {
      const double *Fk = a.F[k];
      for (int e = tid; e < dims[k] * R; e += 64) {
        sA[aoff[k] + e] = a.A[k][e];
        sF[aoff[k] + e] = (Fk != nullptr) ? Fk[e] : 0.0;
      }
    }
  }
  if (tid == 0) {
    sA[kTinyMaxA] = 1.0;
    s_status = 0;
    s_failed = -1;
  }
  __syncthreads();
  // ---- offset tables of the Khatri-Rao halves: WL(a, r) over the modes < n, WR(b, r) over the
  // modes > n, digits of a / b fastest first ----
  if (warp == 0) {
    int left = 1;
#pragma unroll
    for (int n = 0; n < MN; ++n) {
      if (n < N) {
        const int right = P / (left * dims[n]);
        for (int e = lane; e < (left + right) * R; e += 32) {
          const bool isl = e < left * R;
          const int ee = isl ? e : e - left * R;
          const int len = isl ? left : right;
          const int r = ee / len;
          int c = ee - r * len;
          unsigned short o[4] = {kTinyMaxA, kTinyMaxA, kTinyMaxA, kTinyMaxA};
          int j = 0;
#pragma unroll
          for (int k = 0; k < MN; ++k) {
            if (k < N && (isl ? k < n : k > n)) {
              const int c2 = c / dims[k];
              o[j++] = (unsigned short)(aoff[k] + (c - c2 * dims[k]) + dims[k] * r);
              c = c2;
            }
          }
          sTab[n][e] = make_ushort4(o[0], o[1], o[2], o[3]);
        }
        if (lane < left * right) {
          const int bb = lane / left, aa = lane - bb * left;
          sQt[n][lane] = make_ushort4((unsigned short)(aa + left * dims[n] * bb), (unsigned short)aa,
                                      (unsigned short)bb, 0);
        }
        left *= dims[n];
      }
    }
  }
  // Upsilon^(k) = A^(k)T A^(k), sum over i ascending
  if (warp == 1)
  for (int e = lane; e < N * RR; e += 32) {
    const int k = e / RR, rs = e - k * RR, r = rs % R, s = rs / R;
    int ak = 0, Ik = 1;
#pragma unroll
    for (int q = 0; q < MN; ++q)
      if (q == k) {
        ak = aoff[q];
        Ik = dims[q];
      }
    const double *x = sA + ak + Ik * r, *y = sA + ak + Ik * s;
    double g = 0.0;
    for (int i = 0; i < Ik; ++i) g = fma(x[i], y[i], g);
    sU[e] = g;
  }
  __syncthreads();

  double inner_last = 0.0, fa_last = 0.0;
  bool failed_here = false;
  for (int sweep = 0; sweep < a.nsweeps && !failed_here; ++sweep) {
    int left = 1;
#pragma unroll
    for (int n = 0; n < MN; ++n) {
      if (n < N && !failed_here) {
        const int In = dims[n];
        const int right = P / (left * In);
        if (warp == 0) {
          // ---- Khatri-Rao halves (1.0 * a * b * c in digit order, as small_sweep_kernel) ----
          double *sWL = sW, *sWR = sW + left * R;
          for (int e = lane; e < (left + right) * R; e += 32) {
            const ushort4 t = sTab[n][e];
            double w = 1.0;
            w *= sA[t.x];
            w *= sA[t.y];
            w *= sA[t.z];
            sW[e] = w;
          }
          __syncwarp();
          // ---- M(i, r) = sum_{a,b} z(a, i, b) WL(a, r) WR(b, r) (eq:gradEqn) ----
          const int Q = left * right, nout = In * R;
          if (Q <= 1) tiny_mttkrp<1>(sZ, sWL, sWR, sM, sQt[n], Q, left, right, In, invd[n], nout, lane);
          else if (Q <= 2) tiny_mttkrp<2>(sZ, sWL, sWR, sM, sQt[n], Q, left, right, In, invd[n], nout, lane);
          else if (Q <= 4) tiny_mttkrp<4>(sZ, sWL, sWR, sM, sQt[n], Q, left, right, In, invd[n], nout, lane);
          else if (Q <= 8) tiny_mttkrp<8>(sZ, sWL, sWR, sM, sQt[n], Q, left, right, In, invd[n], nout, lane);
          else if (Q <= 16) tiny_mttkrp<16>(sZ, sWL, sWR, sM, sQt[n], Q, left, right, In, invd[n], nout, lane);
          else tiny_mttkrp<32>(sZ, sWL, sWR, sM, sQt[n], Q, left, right, In, invd[n], nout, lane);
        } else {
          // ---- Gamma^(n) = *_{k != n} Upsilon^(k) (eq:Gamma) = L L^T, every lane redundantly in its
          // registers (no pivot broadcast on the chain); lane 0 hands L and 1 / L(j, j) over ----
          double L[R][R], di[R];
          bool ok = true;
#pragma unroll
          for (int c = 0; c < R; ++c)
#pragma unroll
            for (int r = c; r < R; ++r) {
              double g = 1.0;
#pragma unroll
              for (int k = 0; k < MN; ++k)
                if (k < N && k != n) g *= sU[k * RR + r + R * c];
              L[r][c] = g;
            }
#pragma unroll
          for (int j = 0; j < R; ++j) {
            double d = L[j][j];
#pragma unroll
            for (int k = 0; k < j; ++k) d = fma(-L[j][k], L[j][k], d);
            ok = ok && (d > 0.0);
            const double rj = ts_rsqrt(ok ? d : 1.0);
            L[j][j] = d * rj;
            di[j] = rj;
#pragma unroll
            for (int i = j + 1; i < R; ++i) {
              double sv = L[i][j];
#pragma unroll
              for (int k = 0; k < j; ++k) sv = fma(-L[i][k], L[j][k], sv);
              L[i][j] = sv * rj;
            }
          }
          if (lane == 0) {
#pragma unroll
            for (int j = 0; j < R; ++j) {
              sDi[j] = di[j];
#pragma unroll
              for (int i = j; i < R; ++i) sL[i * R + j] = L[i][j];
            }
            if (!ok) {
              s_status = CP_ENOTSPD;
              s_failed = n;
            }
          }
        }
        named_bar_sync(kBarL, 64);  // M (warp 0) and L (warp 1) of mode n are in shared memory
        failed_here = (s_status != 0);
        if (!failed_here) {
          double *An = sA + aoff[n];
          if (warp == 0) {
            // ---- a lane per row: L y = (m + f)^T, L^T x^T = y (eq:relaxinnersolve) ----
            double L[R][R], di[R];
#pragma unroll
            for (int j = 0; j < R; ++j) {
              di[j] = sDi[j];
#pragma unroll
              for (int i = j; i < R; ++i) L[i][j] = sL[i * R + j];
            }
            const double *Fn = sF + aoff[n];
            for (int i = lane; i < In; i += 32) {
              double y[R];
#pragma unroll
              for (int r = 0; r < R; ++r) y[r] = sM[i + In * r] + (anyF ? Fn[i + In * r] : 0.0);
#pragma unroll
              for (int r = 0; r < R; ++r) {
                double bv = y[r];
#pragma unroll
                for (int k = 0; k < r; ++k) bv = fma(-L[r][k], y[k], bv);
                y[r] = bv * di[r];
              }
#pragma unroll
              for (int r = R - 1; r >= 0; --r) {
                double x = y[r];
#pragma unroll
                for (int k = r + 1; k < R; ++k) x = fma(-L[k][r], y[k], x);
                y[r] = x * di[r];
                An[i + In * r] = y[r];
              }
            }
          }
          named_bar_sync(kBarA, 64);  // A^(n) is solved: warp 1 forms its Gram, warp 0 moves on
          if (warp == 1) {
            for (int e = lane; e < RR; e += 32) {
              const int sc = e / R, r = e - sc * R;
              const double *x = An + In * r, *y = An + In * sc;
              double g = 0.0;
              for (int i = 0; i < In; ++i) g = fma(x[i], y[i], g);
              sU[n * RR + e] = g;
            }
            __syncwarp();
          } else if (n == N - 1 && sweep == a.nsweeps - 1) {
            const int nout = In * R;
            double d = 0.0;
            for (int o = lane; o < nout; o += 32) d = fma(sM[o], An[o], d);
            inner_last = warp_sum(d);
          }
        }
        left *= In;
      }
    }
    if (failed_here) break;
    if (sweep == a.nsweeps - 1) {
      // f pieces of the last sweep, before any normalization: ||[[A]]||^2 = 1^T (*_k Upsilon^(k)) 1
      // (warp 1, which holds the Grams) and sum_n <F^(n), A^(n)> (warp 0)
      if (warp == 1) {
        double m2 = 0.0;
        for (int e = lane; e < RR; e += 32) {
          double pr = 1.0;
          for (int k = 0; k < N; ++k) pr *= sU[k * RR + e];
          m2 += pr;
        }
        m2 = warp_sum(m2);
        if (lane == 0) s_model2 = m2;
      } else {
        double fa = 0.0;
        if (anyF)
          for (int e = lane; e < off; e += 32) fa = fma(sF[e], sA[e], fa);
        fa_last = warp_sum(fa);
      }
    }
    if (a.normalize) {
      // eq:ALSnorm after the sweep (cp_normalize_sort with sort = 0): every column
      // scaled to lambda_r = (prod_n ||a_r^(n)||)^(1/N), unless a column norm is zero.  Warp 0
      // scales the factors, then warp 1 recomputes the Grams.
      named_bar_sync(kBarS, 64);
      if (warp == 0) {
        for (int e = lane; e < N * R; e += 32) {
          const int k = e / R, r = e - k * R;
          int ak = 0, Ik = 1;
#pragma unroll
          for (int q = 0; q < MN; ++q)
            if (q == k) {
              ak = aoff[q];
              Ik = dims[q];
            }
          const double *col = sA + ak + Ik * r;
          double ss = 0.0;
          for (int i = 0; i < Ik; ++i) ss = fma(col[i], col[i], ss);
          sNrm[e] = sqrt(ss);
        }
        __syncwarp();
        for (int r = lane; r < R; r += 32) {
          double prod = 1.0;
          int pos = 1;
          for (int k = 0; k < N; ++k) {
            prod *= sNrm[k * R + r];
            pos = pos && (sNrm[k * R + r] > 0.0);
          }
          sLam[r] = pow(prod, 1.0 / (double)N);
          sPos[r] = pos;
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < MN; ++k) {
          if (k < N) {
            double *Ak = sA + aoff[k];
            for (int e = lane; e < dims[k] * R; e += 32) {
              const int r = e / dims[k];
              if (sPos[r]) Ak[e] = sLam[r] * (Ak[e] / sNrm[k * R + r]);
            }
          }
        }
      }
      named_bar_sync(kBarS, 64);
      if (warp == 1) {
        for (int e = lane; e < N * RR; e += 32) {  // the Grams of the normalized factors
          const int k = e / RR, rs = e - k * RR, r = rs % R, s2 = rs / R;
          int ak = 0, Ik = 1;
#pragma unroll
          for (int q = 0; q < MN; ++q)
            if (q == k) {
              ak = aoff[q];
              Ik = dims[q];
            }
          const double *x = sA + ak + Ik * r, *y = sA + ak + Ik * s2;
          double g = 0.0;
          for (int i = 0; i < Ik; ++i) g = fma(x[i], y[i], g);
          sU[e] = g;
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  // ---- write back, f and f~ (readings R6, R5) ----
#pragma unroll
  for (int k = 0; k < kTinyMaxN; ++k)
    if (k < N)
      for (int e = tid; e < dims[k] * R; e += 64) a.A[k][e] = sA[aoff[k] + e];
  if (tid == 0) {
    if (s_status != 0) {
      a.out[0] = nan("");
      a.out[1] = nan("");
      a.out[2] = (double)s_status;
      a.out[3] = (double)s_failed;
    } else {
      const double f = 0.5 * a.normZ2[0] - inner_last + 0.5 * s_model2;
      a.out[0] = f;
      a.out[1] = f - fa_last;
      a.out[2] = 0.0;
      a.out[3] = -1.0;
    }
  }
}

bool tiny_sweep_ok(const cp_shape &s) {
  if (s.R > kTinySweepMaxR || s.N < 2 || s.N > kTinyMaxN) return false;
  int64_t P = 1, sumI = 0, imax = 1;
  for (int k = 0; k < s.N; ++k) {
    if (s.dims[k] > kTinySweepMaxP) return false;
    P *= s.dims[k];
    if (P > kTinySweepMaxP) return false;
    sumI += s.dims[k];
    if (s.dims[k] > imax) imax = s.dims[k];
  }
  if (sumI * s.R > kTinyMaxA || imax * s.R > kTinyMaxM) return false;
  for (int n = 0; n < s.N; ++n) {
    int64_t left = 1, right = 1;
    for (int k = 0; k < n; ++k) left *= s.dims[k];
    for (int k = n + 1; k < s.N; ++k) right *= s.dims[k];
    // one column per lane (the bitwise-equal MTTKRP sum), table rows
    if (left * right > 32 || (left + right) * s.R > kTinyMaxW) return false;
  }
  return true;
}

cudaError_t launch_tiny_sweep(const cp_shape &s, const double *Z, const double *normZ2, double *const *A,
                              const double *const *F, int nsweeps, double *out, cudaStream_t st, bool normalize) {
  SmallSweepArgs a;
  memset(&a, 0, sizeof(a));
  a.normalize = normalize ? 1 : 0;
  a.N = s.N;
  a.R = s.R;
  a.nsweeps = nsweeps;
  a.P = 1;
  for (int k = 0; k < s.N; ++k) {
    a.dims[k] = s.dims[k];
    a.P *= s.dims[k];
    a.A[k] = const_cast<double *>(A[k]);
    a.F[k] = (F != nullptr) ? F[k] : nullptr;
  }
  a.Z = Z;
  a.normZ2 = normZ2;
  a.out = out;
  switch (s.R) {
    case 1: return launch_k(tiny_sweep_kernel<1>, dim3(1), dim3(64), 0, st, a);
    case 2: return launch_k(tiny_sweep_kernel<2>, dim3(1), dim3(64), 0, st, a);
    case 3: return launch_k(tiny_sweep_kernel<3>, dim3(1), dim3(64), 0, st, a);
    case 4: return launch_k(tiny_sweep_kernel<4>, dim3(1), dim3(64), 0, st, a);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace cpk
