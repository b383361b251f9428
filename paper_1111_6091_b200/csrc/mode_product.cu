// mode_product.cu -- n-mode product X = Z x_n U, the restriction Z x_n Phat^T that
// builds coarse-level tensors (eq:ctensor_transformed P:176-180, Alg. 1 step 7 P:273) and the
// interpolation Phat A_c (eq:CGC P:191).  As matrices, X_(n) = U Z_(n); with Z stored mode-1
// fastest this is a strided batched GEMM over the trailing modes:
//   mode 0:      X (J x Q)            = U (J x I1)  * Z (I1 x Q)                  batch 1
//   mode n > 0:  X_b (left x J)       = Z_b (left x I_n) * U^T (I_n x J)          batch b < right
// Two kernels: the fp64 tensor-core (DMMA) GEMM below is the default -- measured 1.5x faster
// than the DFMA register-tiled GEMM (c4a: 26.5 vs 17.1 TFLOP/s, c3: 23 vs 16; profiles/), which
// stays available with CP_MODEPROD_DMMA=0.
#include <cmath>
#include <cstdlib>

#include "cp_internal.cuh"

namespace cpk {

cudaError_t launch_mode_product_dfma(int N, const int64_t *dims, const double *Z, int mode,
                                     const double *U, int64_t J, double *X, cudaStream_t st);

struct GemmArgs {
  int64_t M, N, K, batch;
  const double *A;
  int64_t sam, sak, sab;
  const double *B;
  int64_t sbk, sbn, sbb;
  double *C;
  int64_t scm, scn, scb;
  int swap;  // 1: blockIdx.x indexes n-tiles, blockIdx.y m-tiles (the larger count goes on x)
};

constexpr int BM = 64, BN = 64, BK = 16;

template <bool CM_FAST>  // CM_FAST: C is contiguous along m (threads' fast index -> m)
__global__ void __launch_bounds__(256) gemm_f64_kernel(const GemmArgs g) {
  __shared__ double As[2][BK][BM + 1];
  __shared__ double Bs[2][BK][BN + 1];
  const int t = threadIdx.x;
  const int tx = t & 15, ty = t >> 4;
  const int64_t bm = (int64_t)(g.swap ? blockIdx.y : blockIdx.x) * BM;
  const int64_t bn = (int64_t)(g.swap ? blockIdx.x : blockIdx.y) * BN;
  const int64_t b = blockIdx.z;
  const double *A = g.A + b * g.sab;
  const double *B = g.B + b * g.sbb;
  double *C = g.C + b * g.scb;
  const bool a_mfast = (g.sam == 1);
  const bool b_nfast = (g.sbn == 1);

  double ra[4], rbv[4];
  auto load_tiles = [&](int64_t k0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int mm, kk;
      if (a_mfast) { mm = t & 63; kk = (t >> 6) + 4 * j; }
      else { kk = t & 15; mm = (t >> 4) + 16 * j; }
      const int64_t m = bm + mm, k = k0 + kk;
      ra[j] = (m < g.M && k < g.K) ? __ldg(A + m * g.sam + k * g.sak) : 0.0;
      int nn, kb;
      if (b_nfast) { nn = t & 63; kb = (t >> 6) + 4 * j; }
      else { kb = t & 15; nn = (t >> 4) + 16 * j; }
      const int64_t n = bn + nn, kq = k0 + kb;
      rbv[j] = (n < g.N && kq < g.K) ? __ldg(B + kq * g.sbk + n * g.sbn) : 0.0;
    }
  };
  auto store_tiles = [&](int buf) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int mm, kk;
      if (a_mfast) { mm = t & 63; kk = (t >> 6) + 4 * j; }
      else { kk = t & 15; mm = (t >> 4) + 16 * j; }
      As[buf][kk][mm] = ra[j];
      int nn, kb;
      if (b_nfast) { nn = t & 63; kb = (t >> 6) + 4 * j; }
      else { kb = t & 15; nn = (t >> 4) + 16 * j; }
      Bs[buf][kb][nn] = rbv[j];
    }
  };

  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  const int mi = CM_FAST ? tx : ty;  // thread's m lane
  const int nj = CM_FAST ? ty : tx;  // thread's n lane

  load_tiles(0);
  store_tiles(0);
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = 0; k0 < g.K; k0 += BK) {
    const bool more = (k0 + BK < g.K);
    if (more) load_tiles(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[buf][kk][mi + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[buf][kk][nj + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    if (more) {
      store_tiles(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t m = bm + mi + 16 * i, n = bn + nj + 16 * j;
      if (m < g.M && n < g.N) C[m * g.scm + n * g.scn] = acc[i][j];
    }
}

// ---------------------------------------------------------------------------------------------
// FP64 tensor-core variant (legacy mma.sync.m8n8k4.f64 -> SASS DMMA; tcgen05 has no fp64 kind).
// CTA tile 64 x 128 x 16, 8 warps in a 2 x 4 grid, warp tile 32 x 32 = 4 x 4 m8n8 fragments.
// Operand tiles are kept in shared memory in their global orientation (A_MC: A contiguous
// along m, else along k; B_NC: B contiguous along n, else along k) with padded strides that make
// the fragment reads bank-conflict free (two 128-B wavefronts per 256-B fragment).
constexpr int TBM = 64, TBN = 128, TBK = 16;
// (strides = 4 (mod 16) doubles: a 64-bit shared load is served half-warp by half-warp, and lanes
// (gq, tq) of a half-warp -- gq in 0..3 or 4..7, tq in 0..3 -- then hit the 16 distinct bank pairs
// 4 tq + gq; a stride = 8 (mod 16) collides tq with tq + 2: ncu showed 4 wavefronts per A fragment
// instead of 2 at AMS = 72, profiles/r02g_ncu_gemm_c3.md)
constexpr int AMS = TBM + 4, AKS = TBK + 4, BNS = TBN + 4, BKS = TBK + 4;

__device__ __forceinline__ void dmma_m8n8k4(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <bool A_MC, bool B_NC>
__global__ void __launch_bounds__(256) gemm_dmma_kernel(const GemmArgs g) {
  // double buffer + register prefetch (dynamic shared memory: > 48 KB)
  constexpr int ASZ = A_MC ? TBK * AMS : TBM * AKS, BSZ = B_NC ? TBK * BNS : TBN * BKS;
  extern __shared__ __align__(16) double gsm[];
  double(*As)[ASZ] = reinterpret_cast<double(*)[ASZ]>(gsm);
  double(*Bs)[BSZ] = reinterpret_cast<double(*)[BSZ]>(gsm + 2 * ASZ);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps
  const int gq = lane >> 2, tq = lane & 3;  // fragment coordinates
  const int64_t bm = (int64_t)(g.swap ? blockIdx.y : blockIdx.x) * TBM;
  const int64_t bn = (int64_t)(g.swap ? blockIdx.x : blockIdx.y) * TBN;
  const int64_t b = blockIdx.z;
  const double *A = g.A + b * g.sab;
  const double *B = g.B + b * g.sbb;
  double *C = g.C + b * g.scb;

  double ra[4], rb[8];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int mm, kk;
      if (A_MC) { mm = t & 63; kk = (t >> 6) + 4 * j; }
      else { kk = t & 15; mm = (t >> 4) + 16 * j; }
      const int64_t m = bm + mm, k = k0 + kk;
      ra[j] = (m < g.M && k < g.K) ? __ldg(A + m * g.sam + k * g.sak) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int nn, kk;
      if (B_NC) { nn = t & 127; kk = (t >> 7) + 2 * j; }
      else { kk = t & 15; nn = (t >> 4) + 16 * j; }
      const int64_t n = bn + nn, k = k0 + kk;
      rb[j] = (n < g.N && k < g.K) ? __ldg(B + k * g.sbk + n * g.sbn) : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (A_MC) As[buf][((t >> 6) + 4 * j) * AMS + (t & 63)] = ra[j];
      else As[buf][((t >> 4) + 16 * j) * AKS + (t & 15)] = ra[j];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (B_NC) Bs[buf][((t >> 7) + 2 * j) * BNS + (t & 127)] = rb[j];
      else Bs[buf][((t >> 4) + 16 * j) * BKS + (t & 15)] = rb[j];
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  load(0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = 0; k0 < g.K; k0 += TBK) {
    const bool more = (k0 + TBK < g.K);
    if (more) load(k0 + TBK);
#pragma unroll
    for (int ks = 0; ks < TBK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = wm * 32 + i * 8 + gq, k = ks + tq;
        af[i] = A_MC ? As[buf][k * AMS + m] : As[buf][m * AKS + k];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = wn * 32 + j * 8 + gq, k = ks + tq;
        bf[j] = B_NC ? Bs[buf][k * BNS + n] : Bs[buf][n * BKS + k];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_m8n8k4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (more) {
      // the other buffer was last read in the previous iteration, before that iteration's
      // barrier: store the prefetched tile there, one barrier per k-tile
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t m = bm + wm * 32 + i * 8 + gq;
        const int64_t n = bn + wn * 32 + j * 8 + 2 * tq + h;
        if (m < g.M && n < g.N) C[m * g.scm + n * g.scn] = acc[i][j][h];
      }
}

// ---------------------------------------------------------------------------------------------
// Pipelined FP64 tensor-core GEMM (round 2): the same 64 x 128 CTA tile, 8 warps of 32 x 32 and
// conflict-free padded fragment layouts as gemm_dmma_kernel, but the operand tiles move
// global -> shared with cp.async (16-byte LDGSTS, zero-filled past the matrix edges) through an
// NS-stage ring: NS - 1 k-tiles are in flight while one is multiplied, and the loads never pass
// through registers.  Needs 16-byte pairs along each operand's contiguous dimension (even M, N,
// K, even strides, 16-B aligned bases); launch_mode_product falls back to gemm_dmma_kernel
// otherwise.
__device__ __forceinline__ void cp_async16(void *dst_smem, const void *src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst_smem)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <bool A_MC, bool B_NC, int NS, int TN>
__global__ void __launch_bounds__(256, 2) gemm_dmma_pipe_kernel(const GemmArgs g) {
  // TN: CTA n-tile (128: warp tiles 32 x 32; 64: 32 x 16 -- twice the tiles for the wave
  // quantization of problems with ~1000 tiles, e.g. the c3 restriction)
  constexpr int WF = TN / 32;  // n-fragments (of 8) per warp
  constexpr int BNSx = TN + 4, ASZ = A_MC ? TBK * AMS : TBM * AKS, BSZ = B_NC ? TBK * BNSx : TN * BKS;
  constexpr int BPT = TN * TBK / 2 / 256;  // B pairs per thread
  extern __shared__ __align__(16) double gsm[];
  double *As = gsm, *Bs = gsm + NS * ASZ;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int gq = lane >> 2, tq = lane & 3;
  const int64_t bm = (int64_t)(g.swap ? blockIdx.y : blockIdx.x) * TBM;
  const int64_t bn = (int64_t)(g.swap ? blockIdx.x : blockIdx.y) * TN;
  const int64_t b = blockIdx.z;
  const double *A = g.A + b * g.sab;
  const double *B = g.B + b * g.sbb;
  double *C = g.C + b * g.scb;
  const int64_t nk = (g.K + TBK - 1) / TBK;

  // k-tile kt -> ring slot: A 512 pairs (2 per thread), B TN * 8 pairs (BPT per thread)
  auto issue = [&](int64_t kt) {
    const int slot = (int)(kt % NS);
    const int64_t k0 = kt * TBK;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int pr = t + 256 * j;
      int mm, kk, so;
      if (A_MC) { kk = pr >> 5; mm = (pr & 31) * 2; so = kk * AMS + mm; }
      else { mm = pr >> 3; kk = (pr & 7) * 2; so = mm * AKS + kk; }
      const int64_t m = bm + mm, k = k0 + kk;
      const bool ok = m < g.M && k < g.K;
      cp_async16(As + slot * ASZ + so, ok ? A + m * g.sam + k * g.sak : A, ok ? 16 : 0);
    }
#pragma unroll
    for (int j = 0; j < BPT; ++j) {
      const int pr = t + 256 * j;
      int nn, kk, so;
      if (B_NC) { kk = pr / (TN / 2); nn = (pr % (TN / 2)) * 2; so = kk * BNSx + nn; }
      else { nn = pr >> 3; kk = (pr & 7) * 2; so = nn * BKS + kk; }
      const int64_t n = bn + nn, k = k0 + kk;
      const bool ok = n < g.N && k < g.K;
      cp_async16(Bs + slot * BSZ + so, ok ? B + k * g.sbk + n * g.sbn : B, ok ? 16 : 0);
    }
  };

  double acc[4][WF][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < WF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    if (s < nk) issue(s);
    cp_async_commit();
  }
  for (int64_t kt = 0; kt < nk; ++kt) {
    cp_async_wait<NS - 2>();  // k-tile kt landed (this thread's copies) ...
    __syncthreads();          // ... and everyone's; slot (kt - 1) % NS is free again
    if (kt + NS - 1 < nk) issue(kt + NS - 1);
    cp_async_commit();
    const double *as = As + (int)(kt % NS) * ASZ;
    const double *bs = Bs + (int)(kt % NS) * BSZ;
#pragma unroll
    for (int ks = 0; ks < TBK; ks += 4) {
      double af[4], bf[WF];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = wm * 32 + i * 8 + gq, k = ks + tq;
        af[i] = A_MC ? as[k * AMS + m] : as[m * AKS + k];
      }
#pragma unroll
      for (int j = 0; j < WF; ++j) {
        const int n = wn * (8 * WF) + j * 8 + gq, k = ks + tq;
        bf[j] = B_NC ? bs[k * BNSx + n] : bs[n * BKS + k];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < WF; ++j) dmma_m8n8k4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < WF; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t m = bm + wm * 32 + i * 8 + gq;
        const int64_t n = bn + wn * (8 * WF) + j * 8 + 2 * tq + h;
        if (m < g.M && n < g.N) C[m * g.scm + n * g.scn] = acc[i][j][h];
      }
}

template <bool A_MC, bool B_NC, int NS, int TN>
static size_t dmma_pipe_smem() {
  return NS * sizeof(double) * (size_t)((A_MC ? TBK * AMS : TBM * AKS) + (B_NC ? TBK * (TN + 4) : TN * BKS));
}

template <bool A_MC, bool B_NC, int NS, int TN>
static cudaError_t launch_pipe(const GemmArgs &g, dim3 grid, cudaStream_t st) {
  const size_t sm = dmma_pipe_smem<A_MC, B_NC, NS, TN>();
  if (cudaError_t e = ensure_smem_attr((const void *)gemm_dmma_pipe_kernel<A_MC, B_NC, NS, TN>, (int)sm)) return e;
  gemm_dmma_pipe_kernel<A_MC, B_NC, NS, TN><<<grid, 256, sm, st>>>(g);
  return cudaGetLastError();
}

// the pipelined kernel's 16-byte pair copies are legal for this problem
static bool pipe_ok(const GemmArgs &g, bool a_mc, bool b_nc) {
  auto ev = [](int64_t x) { return (x & 1) == 0; };
  if (!ev(g.M) || !ev(g.N) || !ev(g.K) || !ev(g.sab) || !ev(g.sbb)) return false;
  if (((uintptr_t)g.A % 16) || ((uintptr_t)g.B % 16)) return false;
  if (a_mc ? (g.sam != 1 || !ev(g.sak)) : (g.sak != 1 || !ev(g.sam))) return false;
  if (b_nc ? (g.sbn != 1 || !ev(g.sbk)) : (g.sbk != 1 || !ev(g.sbn))) return false;
  return true;
}

static size_t dmma_smem(bool a_mc, bool b_nc) {
  return 2 * sizeof(double) * (size_t)((a_mc ? TBK * AMS : TBM * AKS) + (b_nc ? TBK * BNS : TBN * BKS));
}
static cudaError_t dmma_attrs() {
  cudaError_t e = ensure_smem_attr((const void *)gemm_dmma_kernel<true, true>, (int)dmma_smem(true, true));
  if (e == cudaSuccess) e = ensure_smem_attr((const void *)gemm_dmma_kernel<true, false>, (int)dmma_smem(true, false));
  return e;
}

cudaError_t launch_mode_product(int N, const int64_t *dims, const double *Z, int mode,
                                const double *U, int64_t J, double *X, cudaStream_t st) {
  if (path_flag("CP_MODEPROD_DMMA", 1)) {
    if (cudaError_t e = dmma_attrs()) return e;
    int64_t left = 1, right = 1;
    for (int k = 0; k < mode; ++k) left *= dims[k];
    for (int k = mode + 1; k < N; ++k) right *= dims[k];
    const int64_t In = dims[mode];
    GemmArgs g;
    bool a_mc, b_nc;
    if (mode == 0) {
      g.M = J; g.N = right; g.K = In; g.batch = 1;
      g.A = U; g.sam = 1; g.sak = J; g.sab = 0;
      g.B = Z; g.sbk = 1; g.sbn = In; g.sbb = 0;
      g.C = X; g.scm = 1; g.scn = J; g.scb = 0;
      a_mc = true; b_nc = false;
    } else {
      g.M = left; g.N = J; g.K = In; g.batch = right;
      g.A = Z; g.sam = 1; g.sak = left; g.sab = left * In;
      g.B = U; g.sbk = J; g.sbn = 1; g.sbb = 0;
      g.C = X; g.scm = 1; g.scn = left; g.scb = left * J;
      a_mc = true; b_nc = true;
    }
    // pipelined kernel, 64 x 128 tiles.  (A 64 x 64 variant, better wave quantization for the
    // ~1000-tile c3 restriction, measured slower: 25.6 vs 28.4 TFLOP/s -- half the DMMAs per
    // fragment load; kept selectable with TN = 64 in launch_pipe.)
    const bool pipe = path_flag("CP_MODEPROD_PIPE", 1) && pipe_ok(g, a_mc, b_nc);
    const int tn = TBN;
    const int64_t gx = (g.M + TBM - 1) / TBM, gy = (g.N + tn - 1) / tn;
    g.swap = (gy > gx) ? 1 : 0;
    const int64_t gbig = g.swap ? gy : gx, gsmall = g.swap ? gx : gy;
    if (gsmall > 65535 || gbig > 0x7fffffff) return cudaErrorInvalidConfiguration;
    for (int64_t b0 = 0; b0 < g.batch; b0 += 65535) {
      GemmArgs gb = g;
      gb.batch = (g.batch - b0) < 65535 ? (g.batch - b0) : 65535;
      gb.A = g.A + b0 * g.sab;
      gb.B = g.B + b0 * g.sbb;
      gb.C = g.C + b0 * g.scb;
      dim3 grid((unsigned)gbig, (unsigned)gsmall, (unsigned)gb.batch);
      cudaError_t e;
      if (pipe) {
        // 4-stage ring when B is n-contiguous, 3 when k-contiguous: <= 113 KB, 2 CTAs/SM
        if (a_mc && b_nc) e = (tn == 64) ? launch_pipe<true, true, 4, 64>(gb, grid, st) : launch_pipe<true, true, 4, 128>(gb, grid, st);
        else e = (tn == 64) ? launch_pipe<true, false, 4, 64>(gb, grid, st) : launch_pipe<true, false, 3, 128>(gb, grid, st);
      } else if (a_mc && b_nc) {
        gemm_dmma_kernel<true, true><<<grid, 256, dmma_smem(true, true), st>>>(gb);
        e = cudaGetLastError();
      } else {
        gemm_dmma_kernel<true, false><<<grid, 256, dmma_smem(true, false), st>>>(gb);
        e = cudaGetLastError();
      }
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  return launch_mode_product_dfma(N, dims, Z, mode, U, J, X, st);
}

cudaError_t launch_mode_product_dfma(int N, const int64_t *dims, const double *Z, int mode,
                                     const double *U, int64_t J, double *X, cudaStream_t st) {
  int64_t left = 1, right = 1;
  for (int k = 0; k < mode; ++k) left *= dims[k];
  for (int k = mode + 1; k < N; ++k) right *= dims[k];
  const int64_t In = dims[mode];
  GemmArgs g;
  if (mode == 0) {
    // X(j, q) = sum_i U(j,i) Z(i,q)
    g.M = J; g.N = right; g.K = In; g.batch = 1;
    g.A = U; g.sam = 1; g.sak = J; g.sab = 0;
    g.B = Z; g.sbk = 1; g.sbn = In; g.sbb = 0;
    g.C = X; g.scm = 1; g.scn = J; g.scb = 0;
  } else {
    // X_b(a, j) = sum_i Z_b(a, i) U(j, i)
    g.M = left; g.N = J; g.K = In; g.batch = right;
    g.A = Z; g.sam = 1; g.sak = left; g.sab = left * In;
    g.B = U; g.sbk = J; g.sbn = 1; g.sbb = 0;
    g.C = X; g.scm = 1; g.scn = left; g.scb = left * J;
  }
  // grid.z is limited to 65535: fold large batches into chunks
  const int64_t gx = (g.M + BM - 1) / BM, gy = (g.N + BN - 1) / BN;
  g.swap = (gy > gx) ? 1 : 0;
  const int64_t gbig = g.swap ? gy : gx, gsmall = g.swap ? gx : gy;
  if (gsmall > 65535 || gbig > 0x7fffffff) return cudaErrorInvalidConfiguration;
  for (int64_t b0 = 0; b0 < g.batch; b0 += 65535) {
    GemmArgs gb = g;
    gb.batch = (g.batch - b0) < 65535 ? (g.batch - b0) : 65535;
    gb.A = g.A + b0 * g.sab;
    gb.B = g.B + b0 * g.sbb;
    gb.C = g.C + b0 * g.scb;
    dim3 grid((unsigned)gbig, (unsigned)gsmall, (unsigned)gb.batch);
    gemm_f64_kernel<true><<<grid, 256, 0, st>>>(gb);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int mode_product_launch_count(int N, const int64_t *dims, int mode) {
  int64_t right = 1;
  for (int k = mode + 1; k < N; ++k) right *= dims[k];
  if (mode == 0) right = 1;
  return (int)((right + 65534) / 65535);
}

}  // namespace cpk
