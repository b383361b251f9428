// stream_kernel.cuh -- the Z-streaming kernel of libcp.so: MTTKRP (eq:gradEqn, eq:Phi,
// P:104-111) and the residual pass of cp_fit (eq:CPfunctional).
//
// Design:
//  * Z is viewed as an I1 x Q column-major matrix (mode-1 fibers are columns).  Every mode's
//    MTTKRP streams Z in that order: a consumer thread owns fixed rows i1 (2 per thread) for
//    the whole pass and keeps R accumulators per row in registers, so the Khatri-Rao row w_q
//    of a column is formed ONCE per column (into shared memory) and broadcast to all rows of
//    the column -- the "reuse along the fast mode" of the north star.
//  * Warp roles (320 threads): warp 8 = TMA producer (one elected lane issues cp.async.bulk
//    copies of the stage's Z columns AND of the factor rows the stage's Khatri-Rao rows need);
//    warp 9 = weight warp (forms w_q[r] = A^(k0)(i_k0, r) * S[r] from the staged rows, S the
//    product of the slowly varying factors); warps 0-7 = consumers (R DFMAs per element).
//    Three mbarrier rings: full (TMA bytes landed), wready (weights formed), empty (consumed).
//  * mode 0 (paper mode 1): the output rows are the owned rows; each column group writes an
//    I1 x R partial, reduced in a fixed order by the next kernel (no atomics).
//  * mode m >= 1: columns are visited with i_m outermost; at the end of each i_m segment the
//    consumers contract their accumulators with A^(1) rows and reduce across the CTA
//    (warp shuffles + shared memory), writing one R-vector partial per (CTA, segment).
#pragma once
#include "cp_internal.cuh"
#if defined(CP_STREAM_TIMING) || defined(CP_CTA_TIMELINE)
#include <cstdio>
#endif

namespace cpk {

// Feature-free instantiations (FEAT = false) of the producer and of stream_mma_kernel: without
// the column-major-factor staging (fcm), the pre-wait Z prefetch and the in-pass completion code
// (sweep_tail, one-launch cp_mttkrp, deferred Gram) the same pass measured 5 us faster on c4a
// (191.3 -> 186.1 us; each feature alone costs 0.9-1.8 us: registers and code around the hot
// loop), so plans that use none of them run the lean kernel (launch_stream).
#define P_FCM(p) (FEAT && (p).fcm != 0)
constexpr int kHdrInts = 16;  // per-stage header: ncols, flags, slot, fcm row offset, digits[kMaxDigits]

// Register budget: up to this many accumulators per thread (V rows x R ranks) the kernel is
// compiled for 2 CTAs/SM (<= 96 registers); above it for 1 CTA/SM.
#ifndef CP_STREAM_2CTA_MAX_VR
#define CP_STREAM_2CTA_MAX_VR 32
#endif

// Shared-memory carve-up of one CTA (all offsets in doubles except the tail).
struct StreamSmem {
  double *zbuf, *abuf, *wbuf, *sbuf, *red, *gjbuf, *sS;
  uint64_t *full, *wready, *empty;
  int *hdr;
};

template <int R, int OP>
__device__ __forceinline__ StreamSmem carve(unsigned char *raw, const StreamPlan &p) {
  constexpr int WSTR = (R % 2 == 0) ? R + 2 : R + 1;
  StreamSmem s;
  s.zbuf = reinterpret_cast<double *>(raw);
  s.abuf = s.zbuf + (size_t)p.nstages * p.zst;
  s.wbuf = s.abuf + (size_t)p.nstages * p.astage;
  s.sbuf = s.wbuf + (size_t)p.nstages * p.cps * p.wstr;
  s.red = s.sbuf + (p.srows ? (size_t)p.nstages * kMaxDigits * p.srs : 0);
  (void)WSTR;
  s.gjbuf = s.red + p.red_doubles;
  s.sS = s.gjbuf + p.gjsm;
  s.full = reinterpret_cast<uint64_t *>(s.sS + 32);
  s.wready = s.full + p.nstages;
  s.empty = s.wready + p.nstages;
  s.hdr = reinterpret_cast<int *>(s.empty + p.nstages);
  return s;
}

// Consumer register tile: RT ranks per thread in RG rank groups.  MTTKRP with R > 12 splits
// the ranks into groups of <= 8 (even RT: 16-B weight loads); R <= 12 and the residual pass
// keep all R ranks in one thread.
template <int R, int OP>
struct StreamTile {
  static constexpr int RG = stream_rg(R, OP);
  static constexpr int RT = stream_rt(R, OP);
};

// Rows owned by consumer unit u of a column block of width Wb: V = 1: {u}; V >= 2: V/2 pairs
// {2u, 2u+1} spaced 2*Wb/V apart (each 16-B load is contiguous across lanes).
template <int V>
__device__ __forceinline__ int row_of(int u, int v, int Wb) {
  if (V == 1) return u;
  return (v >> 1) * ((2 * Wb) / V) + 2 * u + (v & 1);
}
template <int V>
__device__ __forceinline__ void load_rows(const double *zc, int u, int Wb, double (&z)[V]) {
  if (V == 1) {
    z[0] = zc[u];
  } else {
    const int sp = (2 * Wb) / V;
#pragma unroll
    for (int j = 0; j < V / 2; ++j) {
      const double2 a = *reinterpret_cast<const double2 *>(zc + j * sp + 2 * u);
      z[(2 * j) % V] = a.x;
      z[(2 * j + 1) % V] = a.y;
    }
  }
}

// ------------------------------------------------------------------------ producer (warp 8)
// Stage boundaries: a stage never crosses an i_m segment, the CTA's range end, or a wrap of
// the fastest column digit -- so the fastest factor's rows of a stage are contiguous in At
// (one bulk copy) and every slower digit is constant over the stage.
// prefetch (StreamPlan::prefetch, TMA plans): the kernel's predecessor does not write Z, so the Z
// part of the first nstages stages is issued BEFORE the programmatic-dependent-launch wait (the
// HBM latency of the first stages overlaps the predecessor's tail), and their factor rows --
// which the predecessor does write -- after it.  The stage barrier completes only with the
// producer's arrival, which follows both parts.
struct ProducerState {
  int64_t v, seg_left;
  int seg_slot, stage;
  uint32_t eph;
  int B[kMaxDigits];
};
template <int R, int V, bool FEAT = true>
__device__ void produce(const StreamPlan &p, int lane, int64_t v0, int64_t v1, int64_t row0, int Wb,
                        const StreamSmem &sm, bool prefetch = false) {
  const int nd = p.nd;
  const bool has_f0 = (p.ord[0] != p.mode);
  const double *A0 = p.At[p.ord[0]];
  ProducerState st0;
  {
    int64_t t = v0;
#pragma unroll
    for (int j = 0; j < kMaxDigits; ++j) {
      st0.B[j] = 0;
      if (j < nd) {
        st0.B[j] = (int)(t % p.rad[j]);
        t /= p.rad[j];
      }
    }
  }
  st0.seg_left = p.Qn - (v0 % p.Qn);
  st0.seg_slot = 0;
  st0.stage = 0;
  st0.eph = 1;
  st0.v = v0;
#ifdef CP_STREAM_TIMING
  long long tm_wait = 0, tm_n = 0, tm0 = clock64(), tm_pre = 0, tm_issue = 0, tm_post = 0, tm_top = 0;
#endif
  const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
  // part 0: whole stages; 1: Z only (before the wait); 2: the factor rows, header and arrival of
  // the stages part 1 started
  auto run = [&](ProducerState &st, const int part, int max_stages) {
  int (&B)[kMaxDigits] = st.B;
  int64_t &seg_left = st.seg_left, &v = st.v;
  int &seg_slot = st.seg_slot, &stage = st.stage;
  uint32_t &eph = st.eph;
  while (v < v1 && max_stages-- > 0) {
#ifdef CP_STREAM_TIMING
    tm_top = clock64();
#endif
    int64_t lim = (seg_left < v1 - v) ? seg_left : (v1 - v);
    if (lim > p.rad[0] - B[0]) lim = p.rad[0] - B[0];
    const int ncols = (int)(lim < p.cps ? lim : p.cps);
    const bool last = (v + ncols == v1);
    const bool eos = (ncols == seg_left) || last;  // a segment ends, or this CTA's range does
    int64_t q0 = 0;
#pragma unroll
    for (int j = 0; j < kMaxDigits; ++j)
      if (j < nd) q0 += (int64_t)B[j] * p.qsd[j];
#ifdef CP_STREAM_TIMING
    long long tw0 = clock64();
    tm_pre += tw0 - tm_top;
#endif
    if (part != 2) mbar_wait(&sm.empty[stage], eph);
#ifdef CP_STREAM_TIMING
    const long long tw1 = clock64();
    tm_wait += tw1 - tw0;
    ++tm_n;
#endif
    double *zs = sm.zbuf + (size_t)stage * p.zst;
    double *as = sm.abuf + (size_t)stage * p.astage;
    if (V >= 2) {
      int nslow = 0;
      if (p.srows) {
#pragma unroll
        for (int j = 1; j < kMaxDigits; ++j)
          if (j < nd && p.ord[j] != p.mode) ++nslow;
      }
      const bool tstage = p.use_tmap && ncols == p.cps;  // full stage: one tensor-map TMA
      const uint32_t zbytes = tstage ? (uint32_t)(p.zcs * p.cps * 8) : (uint32_t)(ncols * Wb * 8);
      const uint32_t fbytes = (has_f0 ? (P_FCM(p) ? p.fs * p.R * 8 : ncols * p.RS * 8) : 0) +
                              nslow * (P_FCM(p) ? 2 * p.R : p.RS) * 8;
      if (lane == 0) mbar_expect_tx(&sm.full[stage], (part != 2 ? zbytes : 0u) + (part != 1 ? fbytes : 0u));
      __syncwarp();
      if (p.srows && part != 1) {
        // the factor rows of the slow digits (constant over the stage), one copy each (fcm: a
        // {2, R} box of the column-major factor's tensor map: rank r at 2r, p.sstr)
#pragma unroll
        for (int j = 1; j < kMaxDigits; ++j)
          if (j < nd && p.ord[j] != p.mode && lane == j) {
            double *dst = sm.sbuf + ((size_t)stage * kMaxDigits + j) * p.srs;
            if (P_FCM(p))  // (even start row, as for digit 0: the slot holds rows B_j & ~1, +1)
              tma_load_2d(dst, &p.fmap[j], B[j] & ~1, 0, &sm.full[stage]);
            else
              bulk_g2s(dst, p.At[p.ord[j]] + (int64_t)B[j] * p.RS, (uint32_t)(p.RS * 8), &sm.full[stage]);
          }
      }
      // Z columns: q advances by qsd[0] per column within a stage (digit 0 only).  Strided
      // columns are issued by all 32 lanes (one bulk copy per column).
      if (part == 2) {
        // (Z issued by part 1)
      } else if (tstage) {
        if (lane == 0) {
          const int64_t qs = p.qsd[0];
          const int c1 = (int)(q0 % qs), c2 = (int)(q0 / qs);
          if (p.keep_q > 0)
            tma_load_3d_hint(zs, &p.tmap, 0, c1, c2, &sm.full[stage], q0 < p.keep_q ? pol_keep : pol_stream);
          else
            tma_load_3d(zs, &p.tmap, 0, c1, c2, &sm.full[stage]);
        }
      } else if (p.RB == 1 && p.qsd[0] == 1 && p.zcs == 0) {
        if (lane == 0) {
          if (p.keep_q > 0)
            bulk_g2s_hint(zs, p.Z + q0 * p.I1, (uint32_t)(ncols * Wb * 8), &sm.full[stage],
                          q0 < p.keep_q ? pol_keep : pol_stream);
          else
            bulk_g2s(zs, p.Z + q0 * p.I1, (uint32_t)(ncols * Wb * 8), &sm.full[stage]);
        }
      } else {
        const int zstride = p.zcs ? p.zcs : Wb;
        for (int col = lane; col < ncols; col += 32) {
          const int64_t q = q0 + col * p.qsd[0];
          if (p.keep_q > 0)
            bulk_g2s_hint(zs + (size_t)col * zstride, p.Z + q * p.I1 + row0, (uint32_t)(Wb * 8), &sm.full[stage],
                          q < p.keep_q ? pol_keep : pol_stream);
          else
            bulk_g2s(zs + (size_t)col * zstride, p.Z + q * p.I1 + row0, (uint32_t)(Wb * 8), &sm.full[stage]);
        }
      }
      if (part == 1) {
        // (factor rows by part 2, after the wait)
      } else if (has_f0 && P_FCM(p)) {
        // rows B0 .. B0 + fs - 1 of the column-major factor as one {fs, R} box: rank-major
        // [R][fs] in shared memory (rows past I_k zero-filled)
        // (the innermost TMA coordinate must be 16-byte aligned: the box starts at the even row
        // B0 & ~1 and the consumers skip B0 & 1 rows, header word 3)
        if (lane == 31) tma_load_2d(as, &p.fmap[0], B[0] & ~1, 0, &sm.full[stage]);
      } else if (has_f0) {
        if (p.ars == p.RS) {
          if (lane == 31)
            bulk_g2s(as, A0 + (int64_t)B[0] * p.RS, (uint32_t)(ncols * p.RS * 8), &sm.full[stage]);
        } else {  // padded rows (conflict-free B fragments): one copy per factor row
          for (int col = lane; col < ncols; col += 32)
            bulk_g2s(as + (size_t)col * p.ars, A0 + ((int64_t)B[0] + col) * p.RS, (uint32_t)(p.RS * 8),
                     &sm.full[stage]);
        }
      }
      __syncwarp();
    } else {
      // scalar fallback (odd I1: columns are not 16-B aligned): the warp copies elements
      for (int col = 0; col < ncols; ++col) {
        const double *src = p.Z + (q0 + col * p.qsd[0]) * p.I1 + row0;
        for (int i = lane; i < Wb; i += 32) zs[(size_t)col * Wb + i] = __ldg(src + i);
      }
      if (has_f0)
        for (int e = lane; e < ncols * p.RS; e += 32) as[e] = __ldg(A0 + (int64_t)B[0] * p.RS + e);
      __syncwarp();
    }
#ifdef CP_STREAM_TIMING
    const long long tw2 = clock64();
    tm_issue += tw2 - tw1;
#endif
    if (lane == 0 && part != 1) {
      int *h = sm.hdr + stage * kHdrInts;
      h[0] = ncols;
      h[1] = (eos ? 1 : 0) | (last ? 2 : 0);
      h[2] = seg_slot;
      h[3] = B[0] & 1;  // fcm: first staged factor row of the even-aligned box
#pragma unroll
      for (int j = 0; j < kMaxDigits; ++j) h[4 + j] = B[j];
      mbar_arrive(&sm.full[stage]);
    }
    // advance: digit 0 by ncols (at most to its wrap), then carry
    v += ncols;
    B[0] += ncols;
#pragma unroll
    for (int j = 0; j + 1 < kMaxDigits; ++j) {
      if (j + 1 < nd && B[j] >= p.rad[j]) {
        B[j] -= p.rad[j];
        B[j + 1] += 1;
      }
    }
    seg_left -= ncols;
    if (seg_left == 0) {
      seg_left = p.Qn;
      ++seg_slot;
    }
    if (++stage == p.nstages) {
      stage = 0;
      eph ^= 1u;
    }
#ifdef CP_STREAM_TIMING
    tm_post += clock64() - tw2;
#endif
  }
  };
  if (FEAT && prefetch && V >= 2) {
    ProducerState pre = st0;
    run(pre, 1, p.nstages);
    griddep();
    run(st0, 2, p.nstages);
  }
  run(st0, 0, 0x7fffffff);
#ifdef CP_STREAM_TIMING
  if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == 101))
    printf("[cta %d] producer: total %lld wait_empty %lld stages %lld pre %lld issue %lld post %lld\n", blockIdx.x, clock64() - tm0, tm_wait, tm_n, tm_pre, tm_issue, tm_post);
#endif
}

// ------------------------------------------------------------------------ weight warp (warp 9)
// w_q[r] = A^(k0)(i_k0, r) * S[r],  S[r] = prod_{j >= 1, ord[j] != mode} A^(ord[j])(B_j, r).
static __device__ __noinline__ void form_weights(const StreamPlan &p, int lane, const StreamSmem &sm) {
  const int R = p.R;
  const int WSTR = p.wstr;
  if (p.direct_w) return;  // consumers read the staged factor rows themselves
  const int nd = p.nd;
  const bool has_f0 = (p.ord[0] != p.mode);
  int Bc[kMaxDigits];
#pragma unroll
  for (int j = 0; j < kMaxDigits; ++j) Bc[j] = -1;
  int stage = 0;
  uint32_t fph = 0;
#ifdef CP_STREAM_TIMING
  long long tm_wait = 0, tm0 = clock64();
#endif
  for (;;) {
#ifdef CP_STREAM_TIMING
    long long tw0 = clock64();
#endif
    mbar_wait(&sm.full[stage], fph);
#ifdef CP_STREAM_TIMING
    tm_wait += clock64() - tw0;
#endif
    const int *h = sm.hdr + stage * kHdrInts;
    const int ncols = h[0];
    const int flags = h[1];
    bool changed = false;
#pragma unroll
    for (int j = 1; j < kMaxDigits; ++j)
      if (j < nd && h[4 + j] != Bc[j]) changed = true;
    if (changed || Bc[0] == -1) {
      double s = 1.0;
#pragma unroll
      for (int j = 1; j < kMaxDigits; ++j) {
        if (j < nd) {
          Bc[j] = h[4 + j];
          if (p.ord[j] != p.mode && lane < R) s *= __ldg(p.At[p.ord[j]] + (int64_t)Bc[j] * p.RS + lane);
        }
      }
      Bc[0] = 0;
      if (lane < R) sm.sS[lane] = s;
      __syncwarp();
    }
    const double *as = sm.abuf + (size_t)stage * p.astage;
    double *ws = sm.wbuf + (size_t)stage * p.cps * WSTR;
    {
      // lane -> (column, rank) pairs e = lane + 32 i without divisions in the loop
      int col = lane / R, r = lane - (lane / R) * R;
      const int dcol = 32 / R, dr = 32 - (32 / R) * R;
      for (; col < ncols;) {
        ws[col * WSTR + r] = (has_f0 ? as[col * p.ars + r] : 1.0) * sm.sS[r];
        col += dcol;
        r += dr;
        if (r >= R) {
          r -= R;
          ++col;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.wready[stage]);
    if (flags & 2) {
#ifdef CP_STREAM_TIMING
      if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == 101))
        printf("[cta %d] weights: total %lld wait_full %lld\n", blockIdx.x, clock64() - tm0, tm_wait);
#endif
      break;
    }
    if (++stage == p.nstages) {
      stage = 0;
      fph ^= 1u;
    }
  }
}

template <int R, int V, int OP>
__global__ void __launch_bounds__(kStreamThreads, (V * StreamTile<R, OP>::RT <= CP_STREAM_2CTA_MAX_VR ? 2 : 1))
    stream_kernel(const __grid_constant__ StreamPlan p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int WSTR = (R % 2 == 0) ? R + 2 : R + 1;  // weight row stride (even: 16-B aligned)
  const StreamSmem sm = carve<R, OP>(smem_raw, p);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int rb = blockIdx.x % p.RB;
  const int c = blockIdx.x / p.RB;
  const int64_t v0 = (int64_t)c * p.Q / p.Gc;
  const int64_t v1 = (int64_t)(c + 1) * p.Q / p.Gc;
  const int64_t row0 = (int64_t)rb * p.Wmax;
  const int Wb = (int)((p.I1 - row0) < p.Wmax ? (p.I1 - row0) : p.Wmax);  // this block's width

  if (tid == 0) {
    for (int s = 0; s < p.nstages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.wready[s], 1);
      mbar_init(&sm.empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  griddep();  // (PDL) predecessor's At / factor writes visible from here on

  if (warp == kConsumerWarps) {
    produce<R, V>(p, lane, v0, v1, row0, Wb, sm);
    return;
  }
  if (warp == kConsumerWarps + 1) {
    form_weights(p, lane, sm);
    return;
  }

  // ============================ consumer warps ============================
  // Thread tile: V rows x RT ranks (register tiling: each shared-memory load feeds RT or V
  // DFMAs).  Thread t -> (u, g, sl): row unit u (fastest, coalesced), rank group g, column
  // slot sl.  Threads of one column: U * RG; columns per sub-tile: cpt.
  constexpr int RG = StreamTile<R, OP>::RG;
  constexpr int RT = StreamTile<R, OP>::RT;
  const int U = Wb / V;
  const int tpc = U * RG;
  const int cpt = (kConsumers / tpc) > 0 ? (kConsumers / tpc) : 1;
  const int u = tid % U;
  const int g = (tid / U) % RG;
  const int sl = tid / tpc;
  const bool active = sl < cpt;
  const int r0 = g * RT;  // first rank of this thread

  double acc[V][RT];
#pragma unroll
  for (int v = 0; v < V; ++v)
#pragma unroll
    for (int r = 0; r < RT; ++r) acc[v][r] = 0.0;

  double arow[OP == OP_RESID ? V : 1][OP == OP_RESID ? R : 1];
  if (OP == OP_RESID) {
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int r = 0; r < R; ++r)
        arow[v][r] = active ? __ldg(p.At[0] + (row0 + row_of<V>(u, v, Wb)) * p.RS + r) : 0.0;
  }

  int stage = 0;
  uint32_t fph = 0;
#ifdef CP_STREAM_TIMING
  long long tm_wait = 0, tm_loop = 0, tm0 = clock64();
#endif
  for (;;) {
#ifdef CP_STREAM_TIMING
    long long tw0 = clock64();
#endif
    mbar_wait(&sm.wready[stage], fph);
#ifdef CP_STREAM_TIMING
    long long tw1 = clock64();
    tm_wait += tw1 - tw0;
#endif
    // (the weight warp observed full[stage] before arriving on wready: the TMA bytes are visible)
    const int *h = sm.hdr + stage * kHdrInts;
    const int ncols = h[0];
    const int flags = h[1];
    const int slot = h[2];
    const double *zs = sm.zbuf + (size_t)stage * p.zst;
    const double *wsb = sm.wbuf + (size_t)stage * p.cps * WSTR;
    if (active && !(p.dbg & 1)) {
      for (int col = sl; col < ncols; col += cpt) {
        double z[V];
        load_rows<V>(zs + (size_t)col * Wb, u, Wb, z);
        const double *w = wsb + col * WSTR + r0;
        if (OP != OP_RESID) {  // MTTKRP and the Y_L pass: acc += z * w
          double wr[RT];
#pragma unroll
          for (int r = 0; r + 1 < RT; r += 2) {
            const double2 ww = *reinterpret_cast<const double2 *>(w + r);
            wr[r] = ww.x;
            wr[r + 1] = ww.y;
          }
          if (RT & 1) wr[RT - 1] = w[RT - 1];
#pragma unroll
          for (int v = 0; v < V; ++v)
#pragma unroll
            for (int r = 0; r < RT; ++r) acc[v][r] = fma(z[v], wr[r], acc[v][r]);
        } else {
          double x[V];
#pragma unroll
          for (int v = 0; v < V; ++v) x[v] = 0.0;
#pragma unroll
          for (int r = 0; r + 1 < R; r += 2) {
            const double2 ww = *reinterpret_cast<const double2 *>(w + r);
#pragma unroll
            for (int v = 0; v < V; ++v) {
              x[v] = fma(arow[v][r], ww.x, x[v]);
              x[v] = fma(arow[v][r + 1], ww.y, x[v]);
            }
          }
          if (R & 1) {
            const double wl = w[R - 1];
#pragma unroll
            for (int v = 0; v < V; ++v) x[v] = fma(arow[v][R - 1], wl, x[v]);
          }
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const double d = z[v] - x[v];
            acc[v][0] = fma(d, d, acc[v][0]);
          }
        }
      }
    }
    __syncwarp();
#ifdef CP_STREAM_TIMING
    tm_loop += clock64() - tw1;
#endif
    if (lane == 0) mbar_arrive(&sm.empty[stage]);
    if (++stage == p.nstages) {
      stage = 0;
      fph ^= 1u;
    }

    if (OP == OP_YL && (flags & 1)) {
      // ---- end of an i_1 segment: write the I0 x R block of accumulators (slots summed in
      // order through shared memory); a segment shared with a neighbouring CTA goes to this
      // CTA's edge blocks (0: its first segment, 1: its last).  Index arithmetic uses opaque
      // copies so that it stays inside this branch (no hoisted addresses in the loop). ----
      const int Wq = opaque(Wb), uq = opaque(u);
      const int64_t I1q = opaque(p.I1);
      const int64_t s_abs = v0 / p.Qn + slot;
      const bool full = (s_abs * p.Qn >= v0) && ((s_abs + 1) * p.Qn <= v1);
      double *dst = (full ? p.yl + s_abs * I1q * R
                          : p.edge + ((int64_t)blockIdx.x * 2 + (slot == 0 ? 0 : 1)) * I1q * R) +
                    row0 + (int64_t)I1q * r0;
      if (cpt > 1) {
        // slots 1..cpt-1 added to slot 0 in slot order, G slots per round (G regions of
        // Wb x R doubles in the reduction area)
        const int reg = Wq * R;
        const int G = p.red_doubles / reg;
        for (int s1 = 1; s1 < cpt; s1 += G) {
          named_bar_sync(1, kConsumers);
          if (active && sl >= s1 && sl < s1 + G) {
            double *sred = sm.red + (sl - s1) * reg + Wq * r0;
#pragma unroll
            for (int v = 0; v < V; ++v)
#pragma unroll
              for (int r = 0; r < RT; ++r)
                if (r0 + r < R) sred[row_of<V>(uq, v, Wq) + Wq * r] = acc[v][r];
          }
          named_bar_sync(1, kConsumers);
          if (sl == 0) {
            const int n = (cpt - s1 < G) ? cpt - s1 : G;
            for (int k = 0; k < n; ++k) {
              const double *sred = sm.red + k * reg + Wq * r0;
#pragma unroll
              for (int v = 0; v < V; ++v)
#pragma unroll
                for (int r = 0; r < RT; ++r)
                  if (r0 + r < R) acc[v][r] += sred[row_of<V>(uq, v, Wq) + Wq * r];
            }
          }
        }
      }
      if (sl == 0) {
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int r = 0; r < RT; ++r)
            if (r0 + r < R) dst[row_of<V>(uq, v, Wq) + I1q * r] = acc[v][r];
      }
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int r = 0; r < RT; ++r) acc[v][r] = 0.0;
    }
    if (OP == OP_MTTKRP && p.mode != 0 && (flags & 1)) {
      // ---- end of an i_m segment: contract with A^(1) rows and reduce over the CTA ----
      double pr[RT];
#pragma unroll
      for (int r = 0; r < RT; ++r) pr[r] = 0.0;
      if (active) {
#pragma unroll
        const int Wq = opaque(Wb), uq = opaque(u);
        const double *a1b = p.At[0] + row0 * p.RS + r0;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const double *a1 = a1b + (int64_t)row_of<V>(uq, v, Wq) * p.RS;
#pragma unroll
          for (int r = 0; r < RT; ++r)
            if (r0 + r < R) pr[r] = fma(__ldg(a1 + r), acc[v][r], pr[r]);
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int r = 0; r < RT; ++r) acc[v][r] = 0.0;
      if (RG == 1 || U % 32 == 0) {
        // every lane of a warp shares the rank group g: warp shuffles, then one row per warp
#pragma unroll
        for (int r = 0; r < RT; ++r) {
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) pr[r] += __shfl_xor_sync(0xffffffffu, pr[r], off);
        }
        if (lane == 0) {
#pragma unroll
          for (int r = 0; r < RT; ++r) sm.red[warp * RT + r] = pr[r];
        }
        named_bar_sync(1, kConsumers);
        if (tid < R) {
          const int gr = tid / RT, rr = tid - (tid / RT) * RT;
          double sum = 0.0;
          for (int w8 = 0; w8 < kConsumerWarps; ++w8)
            if (((w8 * 32) / U) % RG == gr) sum += sm.red[w8 * RT + rr];
          p.part[((int64_t)blockIdx.x * p.slots + slot) * R + tid] = sum;
        }
      } else {
        // generic: every thread's partial through shared memory, summed in thread order
#pragma unroll
        for (int r = 0; r < RT; ++r) sm.red[tid * RT + r] = pr[r];
        named_bar_sync(1, kConsumers);
        if (tid < R) {
          const int gr = tid / RT, rr = tid - (tid / RT) * RT;
          double sum = 0.0;
          for (int t = 0; t < kConsumers; ++t)
            if ((t / U) % RG == gr) sum += sm.red[t * RT + rr];
          p.part[((int64_t)blockIdx.x * p.slots + slot) * R + tid] = sum;
        }
      }
      named_bar_sync(1, kConsumers);
    }
    if (flags & 2) break;
  }
#ifdef CP_STREAM_TIMING
  if ((tid == 0 || tid == 224) && (blockIdx.x == 0 || blockIdx.x == 101))
    printf("[cta %d tid %d] consumer: total %lld wait_wready %lld loop %lld\n", blockIdx.x, tid, clock64() - tm0, tm_wait, tm_loop);
#endif

  if (OP == OP_MTTKRP && p.mode == 0) {
    // ---- mode 0: write this CTA's I1 x R partial for its row block (slots summed in order) ----
    double *out = p.part + (int64_t)c * p.I1 * R;
    if (cpt > 1) {
      // every consumer is past the ring: reuse it for the slot reduction (slot order, G slots
      // per round)
      const int reg = Wb * R;
      int G = (int)(((int64_t)p.nstages * p.cps * p.Wmax) / reg);
      if (G < 1) G = 1;
      for (int s1 = 1; s1 < cpt; s1 += G) {
        named_bar_sync(1, kConsumers);
        if (active && sl >= s1 && sl < s1 + G) {
          double *sred = sm.zbuf + (sl - s1) * reg + Wb * r0;
#pragma unroll
          for (int v = 0; v < V; ++v)
#pragma unroll
            for (int r = 0; r < RT; ++r)
              if (r0 + r < R) sred[row_of<V>(u, v, Wb) + Wb * r] = acc[v][r];
        }
        named_bar_sync(1, kConsumers);
        if (sl == 0) {
          const int n = (cpt - s1 < G) ? cpt - s1 : G;
          for (int k = 0; k < n; ++k) {
            const double *sred = sm.zbuf + k * reg + Wb * r0;
#pragma unroll
            for (int v = 0; v < V; ++v)
#pragma unroll
              for (int r = 0; r < RT; ++r)
                if (r0 + r < R) acc[v][r] += sred[row_of<V>(u, v, Wb) + Wb * r];
          }
        }
      }
    }
    if (sl == 0) {
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int r = 0; r < RT; ++r)
          if (r0 + r < R) out[row0 + row_of<V>(u, v, Wb) + p.I1 * (r0 + r)] = acc[v][r];
    }
  } else if (OP == OP_RESID) {
    double sacc = 0.0;
#pragma unroll
    for (int v = 0; v < V; ++v) sacc += acc[v][0];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, off);
    if (lane == 0) sm.red[warp] = sacc;
    named_bar_sync(1, kConsumers);
    if (tid == 0) {
      double sum = 0.0;
      for (int w8 = 0; w8 < kConsumerWarps; ++w8) sum += sm.red[w8];
      p.part[blockIdx.x] = sum;
    }
  }
}

template <int R, int V, int OP>
cudaError_t launch_stream_t(const StreamPlan &p, cudaStream_t st) {
  auto kern = stream_kernel<R, V, OP>;
  if (cudaError_t e = ensure_smem_attr((const void *)kern, 200 * 1024)) return e;
  return launch_kc(kPdlStream, kern, dim3(p.Gc * p.RB), dim3(kStreamThreads), (size_t)p.smem_bytes, st, p);
}

}  // namespace cpk
