// stream_mma.cuh -- the Z-streaming MTTKRP / Y_L pass with FP64 tensor-core consumers.
//
// Same pipeline as stream_kernel.cuh (TMA producer warp, weight warp, mbarrier rings, v-order
// odometer, stage boundaries), but the consumers treat each stage as a dense contraction
//     C(rows, ranks) += Z_stage(rows, cols) * W(cols, ranks)
// -- Z(:, i_1, :) A^(2) for the Y_L pass, Z(:, :, j) A^(1) for the mode-2 pass (eq:gradEqn,
// eq:Phi): one mma.sync.m8n8k4.f64 (SASS DMMA) does 8 rows x 8 ranks x 4 columns
// per warp instruction, with the accumulators in registers for the whole pass.
//  * warps: KS k-groups of 8/KS warps; k-group kg takes the k-steps (4 columns) kk = kg mod KS
//    of every stage; warp wi of a group owns m-tiles wi*MT .. wi*MT+MT-1 (8 rows each) and all
//    NT n-tiles (8 ranks each; ranks >= R are masked to zero).
//  * shared memory: Z columns at a padded stride zcs = 8 (mod 16) doubles -> the A-fragment
//    reads (8 rows x 4 columns) take the minimal two 128-B wavefronts; the producer issues one
//    bulk copy per column.  B fragments come from the staged factor rows (direct_w: the
//    Khatri-Rao rows are the factor rows) or from the weight warp's rows.
//  * ragged stages (fewer than 4 columns in a k-step): A and B masked to zero in registers.
//  * residual pass (OP_RESID, cp_fit): the same stages, x = A^(0) W^T on the tensor cores and
//    (z - x)^2 accumulated per thread, one sum per CTA.
//  * epilogues: Y_L pass -- the k-groups' C blocks are summed in group order in shared memory
//    and written as the I0 x R block of the segment (yl, or the CTA's edge block); MTTKRP
//    mode >= 1 -- C contracted with the A^(1) rows, reduced over lanes and warps in a fixed
//    order into one R-vector per (CTA, segment); mode 0 -- the CTA's I1 x R partial.
#pragma once
#include "gamma_job.cuh"
#include "stream_kernel.cuh"

namespace cpk {

__device__ __forceinline__ void dmma_8x8x4(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// k-groups 1..KS-1 add their C blocks into group 0's registers (group order); red holds
// (KS-1) regions of Wb x (8 NT) doubles.  All consumers call it.
template <int NT, int MT>
__device__ __forceinline__ void mma_ksum(double (&acc)[MT][NT][2], double *red, int KS, int kg, int wi, int Wb,
                                         int gq, int tq) {
  if (KS == 1) return;
  const int RP = 8 * NT;
  named_bar_sync(1, kConsumers);
  if (kg > 0) {
    double *dst = red + (size_t)(kg - 1) * Wb * RP;
#pragma unroll
    for (int j = 0; j < MT; ++j) {
      const int m = (wi * MT + j) * 8 + gq;
      if (m < Wb) {
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          dst[(size_t)(n * 8 + 2 * tq) * Wb + m] = acc[j][n][0];
          dst[(size_t)(n * 8 + 2 * tq + 1) * Wb + m] = acc[j][n][1];
        }
      }
    }
  }
  named_bar_sync(1, kConsumers);
  if (kg == 0) {
    for (int g = 1; g < KS; ++g) {
      const double *src = red + (size_t)(g - 1) * Wb * RP;
#pragma unroll
      for (int j = 0; j < MT; ++j) {
        const int m = (wi * MT + j) * 8 + gq;
        if (m < Wb) {
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            acc[j][n][0] += src[(size_t)(n * 8 + 2 * tq) * Wb + m];
            acc[j][n][1] += src[(size_t)(n * 8 + 2 * tq + 1) * Wb + m];
          }
        }
      }
    }
  }
}

// A segment split between CTAs: every contributor, after writing its edge block, takes a ticket
// on the segment's counter; the last one sums the contributors' edge blocks in CTA order into yl
// (the fixed order of yl_fixup_kernel, so results do not depend on which CTA finishes last) and
// resets the counter.  Called by all consumer threads.
__device__ __forceinline__ void yl_complete_segment(const StreamPlan &p, int64_t s, int rb, int64_t row0, int Wb,
                                                 double *scratch) {
  __shared__ int s_last, s_clo, s_chi, s_edclo;
  const int tid = threadIdx.x;
  __threadfence();  // this thread's edge stores before the ticket
  named_bar_sync(1, kConsumers);
  if (tid == 0) {
    const int64_t clo = ((s * p.Qn + 1) * p.Gc - 1) / p.Q;
    const int64_t chi = (((s + 1) * p.Qn) * p.Gc - 1) / p.Q;
    const unsigned old = atomicAdd(p.segcnt + s * p.RB + rb, 1u);
    s_last = (old == (unsigned)(chi - clo)) ? 1 : 0;
    s_clo = (int)clo;
    s_chi = (int)chi;
    s_edclo = ((clo * p.Q) / p.Gc == s * p.Qn) ? 0 : 1;  // s is clo's first segment, else its last
  }
  named_bar_sync(1, kConsumers);
  if (s_last) {
    __threadfence();
    const int R = p.R;
    const int64_t blk = p.I1 * R;
    const int clo = s_clo, chi = s_chi, edclo = s_edclo;
    const int n = Wb * R;
    // 8 elements per thread in flight per contributor (the loop is latency-bound)
    for (int e0 = tid; e0 < n; e0 += 8 * kConsumers) {
      int64_t off[8];
      double acc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * kConsumers;
        const int ec = e < n ? e : 0;
        const int r = ec / Wb, i = ec - (ec / Wb) * Wb;
        off[u] = row0 + i + p.I1 * r;
        acc[u] = 0.0;
      }
      for (int c = clo; c <= chi; ++c) {
        const int ed = (c == clo) ? edclo : 0;
        const double *src = p.edge + (((int64_t)c * p.RB + rb) * 2 + ed) * blk;
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] += __ldcg(src + off[u]);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (e0 + u * kConsumers < n) p.yl[s * blk + off[u]] = acc[u];
    }
    if (tid == 0) p.segcnt[s * p.RB + rb] = 0u;
  }
  (void)scratch;
}

// cp_mttkrp in one launch, modes >= 1 (StreamPlan::Mout): once the CTA has stored the R-vector
// partials of all its segments [s0, s1], it takes a tagged ticket per segment (contributors:
// the CTAs (c, rb), c in [clo, chi]); for every segment where it is the last contributor it sums
// the partials in reduce_entry_part's order (c ascending, then rb) and writes row s of M (one
// warp per segment, lane = rank).  Once per CTA, after the streaming loop: no ticket round trip
// stalls the pipeline.  Called by all consumer threads.
__device__ __forceinline__ void mttkrp_complete_segments(const StreamPlan &p, int64_t v0, int64_t v1) {
  __shared__ int s_last[32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t s0 = v0 / p.Qn, s1 = (v1 - 1) / p.Qn;
  __threadfence();  // the partials' stores before the tickets
  named_bar_sync(1, kConsumers);
  for (int64_t sb = s0; sb <= s1; sb += 32) {
    if (tid < 32) {
      const int64_t s = sb + tid;
      int last = 0;
      if (s <= s1) {
        const int64_t clo = ((s * p.Qn + 1) * p.Gc - 1) / p.Q;
        const int64_t chi = (((s + 1) * p.Qn) * p.Gc - 1) / p.Q;
        last = tagged_arrive(p.tick + s, p.tag, (unsigned)((chi - clo + 1) * p.RB)) ? 1 : 0;
      }
      s_last[tid] = last;
    }
    named_bar_sync(1, kConsumers);
    for (int j = warp; j < 32; j += kConsumerWarps) {
      if (!s_last[j] || lane >= p.R) continue;
      __threadfence();
      const int64_t s = sb + j;
      const int64_t clo = ((s * p.Qn + 1) * p.Gc - 1) / p.Q;
      const int64_t chi = (((s + 1) * p.Qn) * p.Gc - 1) / p.Q;
      double sum = 0.0;
      for (int64_t c = clo; c <= chi; ++c) {
        const int64_t sf = ((c * p.Q) / p.Gc) / p.Qn;
        for (int rb = 0; rb < p.RB; ++rb)
          sum += __ldcg(p.part + ((c * p.RB + rb) * p.slots + (s - sf)) * p.R + lane);
      }
      p.Mout[s + p.In * lane] = sum;
    }
    named_bar_sync(1, kConsumers);
  }
}

// sum of n values at stride, 8 independent accumulators combined in a fixed tree (the order of
// small_kernels.cu sum_strided), L2 loads (the values were written by this launch)
__device__ __forceinline__ double sum_strided_cg(const double *q, int64_t stride, int n) {
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int c = 0;
  for (; c + 8 <= n; c += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] += __ldcg(q + (int64_t)(c + j) * stride);
  }
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (c + j < n) s[j] += __ldcg(q + (int64_t)(c + j) * stride);
  return ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
}

// cp_mttkrp in one launch, mode 0 (StreamPlan::Mout): after the grid barrier every CTA forms the
// entries e in [S b / G, S (b + 1) / G) of M (S = I1 R, column-major like the partials), each as
// 32 chunk sums over the column groups combined in chunk order (reduce_mode0_kernel's order).
// Called by all consumer threads; scratch: 8 x 33 doubles of shared memory.
__device__ __forceinline__ void mttkrp_mode0_slice(const StreamPlan &p, double *scratch) {
  const int tid = threadIdx.x;
  const int64_t S = p.I1 * p.R, G = gridDim.x;
  const int64_t e0 = S * blockIdx.x / G, e1 = S * (blockIdx.x + 1) / G;
  const int ly = tid & 31, j = tid >> 5;  // chunk ly of entry e0 + 8 k + j
  const int c0 = (p.Gc * ly) / 32, c1 = (p.Gc * (ly + 1)) / 32;
  for (int64_t eb = e0; eb < e1; eb += 8) {
    const int64_t e = eb + j;
    scratch[j * 33 + ly] = (e < e1) ? sum_strided_cg(p.part + (int64_t)c0 * S + e, S, c1 - c0) : 0.0;
    named_bar_sync(1, kConsumers);
    if (tid < 8 && eb + tid < e1) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k) t += scratch[tid * 33 + k];
      p.Mout[eb + tid] = t;
    }
    named_bar_sync(1, kConsumers);
  }
}

#ifdef CP_CTA_TIMELINE
__device__ __forceinline__ unsigned long long cta_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

template <int NT, int MT, int OP>
__global__ void __launch_bounds__(kStreamThreads, 2) stream_mma_kernel(const __grid_constant__ StreamPlan p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
#ifdef CP_CTA_TIMELINE
  // timing build only (tools/cta_timeline.py): per-CTA entry, first stage landed, loop end, exit
  unsigned long long tl_enter = cta_gtimer(), tl_first = 0, tl_loop = 0;
  unsigned tl_smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(tl_smid));
#endif
  StreamSmem sm;
  {
    // carve (as carve<R, OP> in stream_kernel.cuh)
    sm.zbuf = reinterpret_cast<double *>(smem_raw);
    sm.abuf = sm.zbuf + (size_t)p.nstages * p.zst;
    sm.wbuf = sm.abuf + (size_t)p.nstages * p.astage;
    sm.sbuf = sm.wbuf + (size_t)p.nstages * p.cps * p.wstr;
    sm.red = sm.sbuf + (p.srows ? (size_t)p.nstages * kMaxDigits * p.srs : 0);
    sm.gjbuf = sm.red + p.red_doubles;
    sm.sS = sm.gjbuf + p.gjsm;
    sm.full = reinterpret_cast<uint64_t *>(sm.sS + 32);
    sm.wready = sm.full + p.nstages;
    sm.empty = sm.wready + p.nstages;
    sm.hdr = reinterpret_cast<int *>(sm.empty + p.nstages);
  }

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int rb = blockIdx.x % p.RB;
  const int c = blockIdx.x / p.RB;
  const int64_t v0 = (int64_t)c * p.Q / p.Gc;
  const int64_t v1 = (int64_t)(c + 1) * p.Q / p.Gc;
  const int64_t row0 = (int64_t)rb * p.Wmax;
  const int Wb = (int)((p.I1 - row0) < p.Wmax ? (p.I1 - row0) : p.Wmax);

  if (tid == 0) {
    for (int s = 0; s < p.nstages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.wready[s], 1);
      mbar_init(&sm.empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  CTL_BEGIN
  griddep();  // (PDL) predecessor's At / factor writes visible from here on
  CTL_AFTER_WAIT
  // one-launch cp_mttkrp, mode 0: CTA 0 claims the grid barrier's words for this launch
  if (OP == OP_MTTKRP && p.mode == 0 && p.Mout != nullptr && blockIdx.x == 0 && tid == 0) grid_claim(p.tick, p.tag);

  if (warp == kConsumerWarps) {
    produce<8, 2>(p, lane, v0, v1, row0, Wb, sm);  // (template args only select the TMA path)
    return;
  }
  if (warp == kConsumerWarps + 1) {
    // weight rows (returns at once when direct_w), then the optional Gamma job of CTA 0
    form_weights(p, lane, sm);
    if (p.gj.on && blockIdx.x == 0) gamma_job_run(p.gj, sm.gjbuf, lane, 32, false);
    return;
  }

  // ============================ consumer warps (tensor cores) ============================
  const int R = p.R;
  const int KS = p.ks;
  const int wpg = kConsumerWarps / KS;  // warps per k-group
  const int kg = warp / wpg, wi = warp - (warp / wpg) * wpg;
  const int gq = lane >> 2, tq = lane & 3;  // fragment coordinates
  const int zcs = p.zcs;
  const int wstride = p.direct_w ? p.ars : p.wstr;
  // B-fragment strides: (column, rank) at col * bcs + rank * brs -- staged rows [col][rank], or
  // (fcm) the rank-major [rank][fs] box of the column-major factor
  const int bcs = p.fcm ? 1 : wstride;
  const int bstage = p.direct_w ? p.astage : p.cps * p.wstr;
  const int arow0 = wi * MT * 8 + gq;  // first A row of this lane (m-tile j adds 8 j)

  double acc[MT][NT][2];
#pragma unroll
  for (int j = 0; j < MT; ++j)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[j][n][0] = acc[j][n][1] = 0.0;

  // B-fragment rank mask (ranks >= R are zero) and the fragment's offset in a staged stage: rank
  // 8n + gq at rank stride fs (fcm) or 1; a masked rank reads rank 0 instead (stays inside the stage of the
  // rank-major fcm layout) and is zeroed in registers
  bool nok[NT];
  int boff[NT];
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    nok[n] = (n * 8 + gq) < R;
    boff[n] = (nok[n] ? n * 8 + gq : 0) * (p.fcm ? p.fs : 1);
  }

  // residual pass (OP_RESID, the mode-0 plan): x(rows, cols) = A^(0)(rows, :) W(cols, :)^T on the
  // tensor cores -- M = rows, N = 8 columns, K = 4 ranks per DMMA; the A fragments (A^(0) rows,
  // constant over the pass) stay in registers; each thread accumulates (z - x)^2
  constexpr int KR = (OP == OP_RESID) ? 2 * NT : 1;  // k-steps of 4 ranks
  double aR[OP == OP_RESID ? MT : 1][KR];
  double racc = 0.0;
  if (OP == OP_RESID) {
#pragma unroll
    for (int j = 0; j < MT; ++j)
#pragma unroll
      for (int kk = 0; kk < KR; ++kk) {
        const int m = arow0 + 8 * j, rk = 4 * kk + tq;
        aR[j][kk] = (m < Wb && rk < R) ? __ldg(p.At[0] + (row0 + m) * p.RS + rk) : 0.0;
      }
  }

  int stage = 0;
  uint32_t fph = 0;
  for (;;) {
    mbar_wait(p.direct_w ? &sm.full[stage] : &sm.wready[stage], fph);
#ifdef CP_CTA_TIMELINE
    if (tl_first == 0) tl_first = cta_gtimer();
#endif
    const int *h = sm.hdr + stage * kHdrInts;
    const int ncols = h[0];
    const int flags = h[1];
    const int slot = h[2];
    const double *zs = sm.zbuf + (size_t)stage * p.zst + arow0;
    const double *ws = (p.direct_w ? sm.abuf : sm.wbuf) + (size_t)stage * bstage + (p.fcm ? h[3] : 0);
    // Khatri-Rao rows = staged factor rows x S, S = product of the slow digits' rows (staged by
    // the producer; S = 1 when there are none)
    double sl[NT];
#pragma unroll
    for (int n = 0; n < NT; ++n) sl[n] = 1.0;
    if (p.srows) {
#pragma unroll
      for (int j = 1; j < kMaxDigits; ++j) {
        if (j < p.nd && p.ord[j] != p.mode) {
          const double *sr = sm.sbuf + ((size_t)stage * kMaxDigits + j) * p.srs + gq * p.sstr + (p.fcm ? (h[4 + j] & 1) : 0);
#pragma unroll
          for (int n = 0; n < NT; ++n)
            if (nok[n]) sl[n] *= sr[8 * n * p.sstr];
        }
      }
    }
    if (OP == OP_RESID) {
      // k-group kg takes the 8-column tiles nc = kg (mod KS) of the stage
      double slr[KR];
#pragma unroll
      for (int kk = 0; kk < KR; ++kk) slr[kk] = (4 * kk + tq < R) ? 1.0 : 0.0;
      if (p.srows) {
#pragma unroll
        for (int j = 1; j < kMaxDigits; ++j) {
          if (j < p.nd && p.ord[j] != p.mode) {
            const double *sr = sm.sbuf + ((size_t)stage * kMaxDigits + j) * p.srs;
#pragma unroll
            for (int kk = 0; kk < KR; ++kk)
              if (4 * kk + tq < R) slr[kk] *= sr[4 * kk + tq];
          }
        }
      }
      const double *zb = sm.zbuf + (size_t)stage * p.zst;
      const double *wbase = (p.direct_w ? sm.abuf : sm.wbuf) + (size_t)stage * bstage;
      for (int nc = kg; nc * 8 < ncols; nc += KS) {
        const int col = nc * 8 + gq;
        const double *wb = wbase + (col < ncols ? col : 0) * wstride;
        double b[KR];
#pragma unroll
        // (a select, not a multiply by the 0/1 mask: the padding ranks >= R of a staged row are
        // never written and may hold NaN bit patterns)
        for (int kk = 0; kk < KR; ++kk) b[kk] = (col < ncols && 4 * kk + tq < R) ? wb[4 * kk + tq] * slr[kk] : 0.0;
        const int c = nc * 8 + 2 * tq;
#pragma unroll
        for (int j = 0; j < MT; ++j) {
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int kk = 0; kk < KR; ++kk) dmma_8x8x4(c0, c1, aR[j][kk], b[kk]);
          const int m = arow0 + 8 * j;
          if (m < Wb) {
            if (c < ncols) {
              const double d = zb[(size_t)c * zcs + m] - c0;
              racc = fma(d, d, racc);
            }
            if (c + 1 < ncols) {
              const double d = zb[(size_t)(c + 1) * zcs + m] - c1;
              racc = fma(d, d, racc);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[stage]);
      if (++stage == p.nstages) {
        stage = 0;
        fph ^= 1u;
      }
      if (flags & 2) break;
      continue;
    }
    // full k-steps (4 landed columns): only the rank mask applies
    int k0 = 4 * kg;
    for (; k0 + 4 <= ncols; k0 += 4 * KS) {
      const int col = k0 + tq;
      const double *za = zs + col * zcs;
      const double *wb = ws + col * bcs;
      double a[MT], b[NT];
#pragma unroll
      for (int j = 0; j < MT; ++j) a[j] = za[8 * j];
#pragma unroll
      for (int n = 0; n < NT; ++n) b[n] = wb[boff[n]];
#pragma unroll
      for (int n = 0; n < NT; ++n) b[n] = nok[n] ? b[n] * sl[n] : 0.0;
#pragma unroll
      for (int j = 0; j < MT; ++j)
#pragma unroll
        for (int n = 0; n < NT; ++n) dmma_8x8x4(acc[j][n][0], acc[j][n][1], a[j], b[n]);
    }
    if (k0 < ncols) {
      // ragged last k-step: columns >= ncols read column 0 of the stage (always landed) and
      // are zeroed in registers (branch-free)
      const int col = k0 + tq;
      const bool ok = col < ncols;
      const int colc = ok ? col : 0;
      const double *za = zs + colc * zcs;
      const double *wb = ws + colc * bcs;
      double a[MT], b[NT];
#pragma unroll
      for (int j = 0; j < MT; ++j) a[j] = za[8 * j];
#pragma unroll
      for (int n = 0; n < NT; ++n) b[n] = wb[boff[n]];
#pragma unroll
      for (int j = 0; j < MT; ++j) a[j] = ok ? a[j] : 0.0;
#pragma unroll
      for (int n = 0; n < NT; ++n) b[n] = (ok && nok[n]) ? b[n] * sl[n] : 0.0;
#pragma unroll
      for (int j = 0; j < MT; ++j)
#pragma unroll
        for (int n = 0; n < NT; ++n) dmma_8x8x4(acc[j][n][0], acc[j][n][1], a[j], b[n]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[stage]);
    if (++stage == p.nstages) {
      stage = 0;
      fph ^= 1u;
    }

    if (OP == OP_YL && (flags & 1)) {
      // ---- end of an i_1 segment: the CTA's I0-block x R block of Y_L(:, i_1, :) ----
      const int Wq = opaque(Wb);
      const int64_t I1q = opaque(p.I1);
      mma_ksum<NT, MT>(acc, sm.red, KS, kg, wi, Wq, gq, tq);
      const int64_t s_abs = v0 / p.Qn + slot;
      const bool full = (s_abs * p.Qn >= v0) && ((s_abs + 1) * p.Qn <= v1);
      if (kg == 0) {
        double *dst = (full ? p.yl + s_abs * I1q * R
                            : p.edge + ((int64_t)blockIdx.x * 2 + (slot == 0 ? 0 : 1)) * I1q * R) +
                      row0;
#pragma unroll
        for (int j = 0; j < MT; ++j) {
          const int m = arow0 + 8 * j;
          if (m < Wq) {
#pragma unroll
            for (int n = 0; n < NT; ++n) {
              const int r = n * 8 + 2 * tq;
              if (r < R) dst[m + I1q * r] = acc[j][n][0];
              if (r + 1 < R) dst[m + I1q * (r + 1)] = acc[j][n][1];
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < MT; ++j)
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[j][n][0] = acc[j][n][1] = 0.0;
      if (!full && p.segcnt != nullptr) yl_complete_segment(p, s_abs, rb, row0, Wq, sm.red);
    }
    if (OP == OP_MTTKRP && p.mode != 0 && (flags & 1)) {
      // ---- end of an i_m segment: contract with the A^(1) rows, reduce lanes and warps ----
      const int Wq = opaque(Wb);
      double pr[NT][2];
#pragma unroll
      for (int n = 0; n < NT; ++n) pr[n][0] = pr[n][1] = 0.0;
      // A^(1) rows: the row-major copy, or (fcm) the caller's column-major factor
      const double *a1b = p.fcm ? p.Af[0] + row0 : p.At[0] + row0 * p.RS;
      const int64_t a1rs = p.fcm ? 1 : p.RS, a1cs = p.fcm ? p.dims[0] : 1;
#pragma unroll
      for (int j = 0; j < MT; ++j) {
        const int m = arow0 + 8 * j;
        if (m < Wq) {
          const double *a1 = a1b + (int64_t)m * a1rs;
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            const int r = n * 8 + 2 * tq;
            if (r < R) pr[n][0] = fma(__ldg(a1 + r * a1cs), acc[j][n][0], pr[n][0]);
            if (r + 1 < R) pr[n][1] = fma(__ldg(a1 + (r + 1) * a1cs), acc[j][n][1], pr[n][1]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < MT; ++j)
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[j][n][0] = acc[j][n][1] = 0.0;
      // lanes sharing tq hold the same ranks: fixed xor tree over gq
#pragma unroll
      for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
          for (int off = 4; off < 32; off <<= 1) pr[n][hh] += __shfl_xor_sync(0xffffffffu, pr[n][hh], off);
      if (gq == 0) {
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          sm.red[warp * 8 * NT + n * 8 + 2 * tq] = pr[n][0];
          sm.red[warp * 8 * NT + n * 8 + 2 * tq + 1] = pr[n][1];
        }
      }
      named_bar_sync(1, kConsumers);
      if (tid < R) {
        double sum = 0.0;
        for (int w8 = 0; w8 < kConsumerWarps; ++w8) sum += sm.red[w8 * 8 * NT + tid];
        p.part[((int64_t)blockIdx.x * p.slots + slot) * R + tid] = sum;
      }
      named_bar_sync(1, kConsumers);
    }
    if (flags & 2) break;
  }
#ifdef CP_CTA_TIMELINE
  tl_loop = cta_gtimer();
#endif
  if (OP == OP_MTTKRP && p.mode != 0 && p.Mout != nullptr) mttkrp_complete_segments(p, v0, v1);

  if (OP == OP_RESID) {
    // ---- this CTA's sum of (z - x)^2: lanes, then warps in order ----
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) racc += __shfl_xor_sync(0xffffffffu, racc, off);
    if (lane == 0) sm.red[warp] = racc;
    named_bar_sync(1, kConsumers);
    if (tid == 0) {
      double sum = 0.0;
      for (int w8 = 0; w8 < kConsumerWarps; ++w8) sum += sm.red[w8];
      p.part[blockIdx.x] = sum;
    }
  }
  if (OP == OP_MTTKRP && p.mode == 0) {
    // ---- mode 0: this CTA's I1 x R partial for its row block (k-groups summed in order
    // through the Z ring, which every consumer is done with) ----
    mma_ksum<NT, MT>(acc, sm.zbuf, KS, kg, wi, Wb, gq, tq);
    if (kg == 0) {
      double *out = p.part + (int64_t)c * p.I1 * R + row0;
#pragma unroll
      for (int j = 0; j < MT; ++j) {
        const int m = arow0 + 8 * j;
        if (m < Wb) {
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            const int r = n * 8 + 2 * tq;
            if (r < R) out[m + p.I1 * r] = acc[j][n][0];
            if (r + 1 < R) out[m + p.I1 * (r + 1)] = acc[j][n][1];
          }
        }
      }
    }
    if (p.Mout != nullptr) {
      // one launch: every CTA's partial stored -> grid barrier -> this CTA's slice of M
      __threadfence();
      named_bar_sync(1, kConsumers);
      if (tid == 0) grid_barrier(p.tick, p.tag, gridDim.x);
      named_bar_sync(1, kConsumers);
      mttkrp_mode0_slice(p, sm.zbuf);
      if (tid == 0) grid_depart(p.tick, p.tag, gridDim.x);
    }
  }
#ifdef CP_CTA_TIMELINE_STREAM
  if (tid == 0)
    printf("CTL %d %d %d %u %llu %llu %llu %llu\n", OP, p.mode, blockIdx.x, tl_smid, tl_enter, tl_first, tl_loop,
           cta_gtimer());
#endif
#ifdef CP_CTA_TIMELINE_STREAM
  CTL_END(OP == OP_YL ? "streamYL" : (OP == OP_RESID ? "streamRES" : (p.mode == 0 ? "streamM0" : "streamMn")))
#endif
}

template <int NT, int MT, int OP>
cudaError_t launch_stream_mma_t(const StreamPlan &p, cudaStream_t st) {
  auto kern = stream_mma_kernel<NT, MT, OP>;
  if (cudaError_t e = ensure_smem_attr((const void *)kern, 200 * 1024)) return e;
  return launch_kc(kPdlStream, kern, dim3(p.Gc * p.RB), dim3(kStreamThreads), (size_t)p.smem_bytes, st, p);
}

}  // namespace cpk
