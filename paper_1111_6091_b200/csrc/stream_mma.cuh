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
//  * shared memory: Z columns at a padded stride zcs = 8 (mod 16) doubles (A-fragment reads of 8
//    rows x 4 columns: 4 wavefronts; = 4 (mod 16) would give 2, see plan_mma); the producer issues one
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
#ifdef CP_TAIL_TIMING
#include <cstdio>
#endif
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

// Sums of three values over the 256 consumer threads (warp xor trees, then the 8 warp sums in a
// fixed order; sred: 24 doubles).  Every consumer calls it; all of them get the sums.
__device__ __forceinline__ void consumer_sum3(double &a, double &b, double &c, double *sred) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, off);
    b += __shfl_xor_sync(0xffffffffu, b, off);
    c += __shfl_xor_sync(0xffffffffu, c, off);
  }
  named_bar_sync(1, kConsumers);
  if (lane == 0) {
    sred[w] = a;
    sred[8 + w] = b;
    sred[16 + w] = c;
  }
  named_bar_sync(1, kConsumers);
  a = ((sred[0] + sred[1]) + (sred[2] + sred[3])) + ((sred[4] + sred[5]) + (sred[6] + sred[7]));
  b = ((sred[8] + sred[9]) + (sred[10] + sred[11])) + ((sred[12] + sred[13]) + (sred[14] + sred[15]));
  c = ((sred[16] + sred[17]) + (sred[18] + sred[19])) + ((sred[20] + sred[21]) + (sred[22] + sred[23]));
}

// C(8 i + m, 8 j + n) += sum_k X(k, 8 i + m) X(k, 8 j + n) over rows k in [r0, r1) of the row-major
// X (stride RS, columns < R): one DMMA per (i, j) and 4 rows; lane (gq, tq) holds X(k0 + tq, 8 i + gq)
// -- both the A and the B fragment.  L2 loads (the rows may have been written by this launch).
template <int NT>
__device__ __forceinline__ void gram_rows_dmma(double (&c)[NT][NT][2], const double *X, int RS, int R, int64_t r0,
                                               int64_t r1, int lane) {
  const int gq = lane >> 2, tq = lane & 3;
  constexpr int KB = (NT <= 2) ? 8 : 4;  // k-steps loaded per batch
  for (int64_t k0 = r0; k0 < r1; k0 += 4 * KB) {
    double xf[KB][NT];
#pragma unroll
    for (int u = 0; u < KB; ++u) {
      const int64_t row = k0 + 4 * u + tq;
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        const int col = 8 * i + gq;
        xf[u][i] = (row < r1 && col < R) ? __ldcg(X + row * RS + col) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < KB; ++u)
#pragma unroll
      for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma_8x8x4(c[i][j][0], c[i][j][1], xf[u][i], xf[u][j]);
  }
}

// The Gram a tail solve deferred (GammaJob::gram_rows): one warp (the idle weight warp of CTA 0)
// forms Upsilon^(gram_mode) over all rows in row order and writes the total to ups.
template <int NT>
__device__ __noinline__ void gram_rows_warp(const GammaJob &g, int lane) {
  if (g.status[0] != 0.0) return;
  const int gq = lane >> 2, tq = lane & 3, R = g.R;
  double c[NT][NT][2];
#pragma unroll
  for (int i = 0; i < NT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) c[i][j][0] = c[i][j][1] = 0.0;
  gram_rows_dmma<NT>(c, g.gram_At, g.gram_RS, R, 0, g.gram_rows, lane);
  double *u = g.ups + (int64_t)g.gram_mode * R * R;
#pragma unroll
  for (int i = 0; i < NT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int r = 8 * i + gq, q = 8 * j + 2 * tq;
      if (r < R && q < R) u[q * R + r] = c[i][j][0];
      if (r < R && q + 1 < R) u[(q + 1) * R + r] = c[i][j][1];
    }
  __syncwarp();
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// The sweep's last solve + finalize inside the mode-2 pass (TailSolve, cp_internal.cuh): called
// by all consumer threads after the streaming loop; scr = the Z ring, which every consumer is
// done with.  The chain after the last stage is a handful of L2 round trips:
//  1. warp 0 takes the segments' tickets (u32 counters zeroed by prep and reset by their last
//     arrival) while the other warps acquire the Gamma job's flag (CTA 0's weight warp set it at
//     the start of the pass) and stage L^{-1};
//  2. per segment s where this CTA arrived last: one warp sums the partials (reduce_entry_part's
//     order), b = m + f, y = L^{-1} b, x = L^{-T} y with the lane's row / column of L^{-1} and one
//     shuffle per term (the term order of solve_kernel_t: the same x bitwise), stores the row of
//     A^(2), At^(2) and the row's <M,A>, <F,A>;
//  3. grid ticket: the last CTA forms Upsilon^(2) = At^T At on the tensor cores straight from L2
//     (warp w: rows [w, w + 1) In / 8 in k-steps of 4, A and B fragments are the same values; the
//     warps' tiles summed in warp order), sums the row dots and the earlier modes' <F,A>
//     partials in a fixed order and writes f, f~, status.  Which CTA runs a step varies from run
//     to run; what it computes does not.
template <int NT>
__device__ __noinline__ void sweep_tail(const StreamPlan &p, int64_t v0, int64_t v1, double *scr) {
  __shared__ int s_last[32], s_clo[32], s_nc[32];
  __shared__ int s_fin, s_live;
  const TailSolve &t = p.tail;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int R = p.R, RR = R * R, LS = R + 1, RS = p.RS;
  constexpr int RP = 8 * NT;
  const int64_t In = p.In;
  const int64_t s0 = v0 / p.Qn, s1 = (v1 - 1) / p.Qn;  // host: s1 - s0 < 32 (slots <= 32)
  double *sLi = scr, *sred = scr + R * LS, *tiles = scr + sweep_tail_fixed_doubles(R);
#ifdef CP_TAIL_TIMING
  unsigned long long tt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define TAIL_T(k) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt[k])); }
#else
#define TAIL_T(k)
#endif
  TAIL_T(0)
  __threadfence();  // the partials' stores before the tickets
  named_bar_sync(1, kConsumers);
  TAIL_T(1)
  if (warp == 0) {
    const int64_t s = s0 + lane;
    int last = 0;
    if (s <= s1) {
      const int64_t clo = ((s * p.Qn + 1) * p.Gc - 1) / p.Q;
      const int64_t chi = (((s + 1) * p.Qn) * p.Gc - 1) / p.Q;
      const unsigned n = (unsigned)((chi - clo + 1) * p.RB);
      s_clo[lane] = (int)clo;
      s_nc[lane] = (int)(chi - clo + 1);
      if (atomicAdd(t.segtick + s, 1u) == n - 1) {
        t.segtick[s] = 0u;
        last = 1;
      }
    }
    s_last[lane] = last;
    // (acquire for the whole CTA: this fence, then the barrier, order the other contributors'
    // partials before every consumer's L2 loads below)
    __threadfence();
  } else {
    const long long t0 = clock64();
    while (ld_acquire_u32(t.gjflag) != 1u) {
      if (clock64() - t0 > 20000000000LL) __trap();
    }
    if (tid == 32) s_live = (__ldcg(t.status) == 0.0) ? 1 : 0;
    for (int e = tid - 32; e < RR; e += kConsumers - 32) sLi[(e / R) * LS + (e % R)] = __ldcg(t.linv + e);
  }
  named_bar_sync(1, kConsumers);
  TAIL_T(2)
  const bool live = s_live != 0;
  for (int j = warp; j < 32; j += kConsumerWarps) {
    if (!s_last[j] || !live) continue;
    const int64_t s = s0 + j;
    const int clo = s_clo[j], nc = s_nc[j];
    const bool on = lane < R;
    const int lr = on ? lane : 0;
    // contributor c's slot of segment s: 32 contributors' offsets formed lane-parallel, then one
    // shuffle each (c ascending, then rb: reduce_entry_part's order)
    const double f = (t.F != nullptr) ? __ldg(t.F + s + In * lr) : 0.0;
    double m = 0.0;
    for (int cb = 0; cb < nc; cb += 32) {
      int64_t myoff = 0;
      if (cb + lane < nc) {
        const int64_t c = clo + cb + lane;
        const int64_t sf = ((c * p.Q) / p.Gc) / p.Qn;
        myoff = ((c * p.RB) * p.slots + (s - sf)) * R;
      }
      const int ncb = (nc - cb) < 32 ? (nc - cb) : 32;
      for (int cc = 0; cc < ncb; ++cc) {
        const int64_t off = __shfl_sync(0xffffffffu, myoff, cc);
        for (int rb = 0; rb < p.RB; ++rb) m += __ldcg(p.part + off + (int64_t)rb * p.slots * R + lr);
      }
    }
    const double b = m + f;
    // y = L^{-1} b, x = L^{-T} y: lane r walks row r / column r of L^{-1}; every term's shuffle
    // and shared-memory load is independent of the fma chain (unrolled by 8: in flight together)
    double y = 0.0, x = 0.0;
    const double *lrow = sLi + lr * LS, *lcol = sLi + lr;
#pragma unroll
    for (int k8 = 0; k8 < RP; k8 += 8) {
      if (k8 < R) {
        double l8[8], b8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = k8 + u;
          l8[u] = (k <= lr && k < R) ? lrow[k] : 0.0;
          b8[u] = __shfl_sync(0xffffffffu, b, k & 31);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (k8 + u <= lr && k8 + u < R) y = fma(l8[u], b8[u], y);
      }
    }
#pragma unroll
    for (int k8 = 0; k8 < RP; k8 += 8) {
      if (k8 < R) {
        double l8[8], y8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = k8 + u;
          l8[u] = (k >= lr && k < R) ? lcol[k * LS] : 0.0;
          y8[u] = __shfl_sync(0xffffffffu, y, k & 31);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (k8 + u >= lr && k8 + u < R) x = fma(l8[u], y8[u], x);
      }
    }
    if (on) {
      t.A[s + In * lane] = x;
      t.At[s * RS + lane] = x;
    }
    double dm = on ? m * x : 0.0, df = on ? f * x : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      dm += __shfl_xor_sync(0xffffffffu, dm, off);
      df += __shfl_xor_sync(0xffffffffu, df, off);
    }
    if (lane == 0) {
      t.rowdot[s] = dm;
      t.rowdot[In + s] = df;
    }
  }
  // ---- grid ticket: the last CTA finalizes ----
  TAIL_T(3)
  __threadfence();
  named_bar_sync(1, kConsumers);
  if (tid == 0) s_fin = (atomicAdd(t.gtick, 1u) == gridDim.x - 1) ? 1 : 0;
  named_bar_sync(1, kConsumers);
  TAIL_T(4)
#ifdef CP_TAIL_TIMING
  if (tid == 0 && (blockIdx.x % 37 == 0) && !s_fin)
    printf("TAIL cta %d: t0 %llu fence+bar %llu tick/flag %llu solve %llu gtick %llu\n", (int)blockIdx.x,
           tt[0], tt[1] - tt[0], tt[2] - tt[1], tt[3] - tt[2], tt[4] - tt[3]);
#endif
  if (!s_fin) return;
  __threadfence();
  if (tid == 0) {  // every CTA is past its flag wait and its arrival: reset for the next launch
    *t.gtick = 0u;
    *t.gjflag = 0u;
  }
  if (!t.fin) return;  // (Upsilon^(2) is formed by the next sweep's Gamma^(0) job; no f this sweep)
  const double st = __ldcg(t.status);
  if (st != 0.0) {
    if (tid == 0) {
      t.out[0] = nan("");
      t.out[1] = nan("");
      t.out[2] = st;
      t.out[3] = __ldcg(t.status + 1);
    }
    return;
  }
  // row dots and the earlier modes' <F,A> partials (loads in flight during the Gram)
  double in = 0.0, fl = 0.0;
  for (int64_t i = tid; i < In; i += kConsumers) {
    in += __ldcg(t.rowdot + i);
    fl += __ldcg(t.rowdot + In + i);
  }
  for (int n = 0; n < 2; ++n)
    for (int c = tid; c < t.nsolve[n]; c += kConsumers) fl += __ldcg(t.dotF + (int64_t)n * t.dot_stride + c);
  // Upsilon^(2) = At^T At on the tensor cores: warp w takes the rows [w, w + 1) rpw
  {
    const int gq = lane >> 2, tq = lane & 3;
    const int64_t rpw = (((In + kConsumerWarps - 1) / kConsumerWarps) + 3) & ~(int64_t)3;
    const int64_t r0 = warp * rpw, r1 = (r0 + rpw < In) ? r0 + rpw : In;
    double c[NT][NT][2];
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) c[i][j][0] = c[i][j][1] = 0.0;
    gram_rows_dmma<NT>(c, t.At, RS, R, r0, r1, lane);
    double *tw = tiles + (size_t)warp * RP * RP;
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        tw[(8 * i + gq) * RP + 8 * j + 2 * tq] = c[i][j][0];
        tw[(8 * i + gq) * RP + 8 * j + 2 * tq + 1] = c[i][j][1];
      }
  }
  TAIL_T(5)
  named_bar_sync(1, kConsumers);
  double m2 = 0.0;
  for (int e = tid; e < RR; e += kConsumers) {
    const int r = e % R, q = e / R;
    double u = 0.0;
#pragma unroll
    for (int w8 = 0; w8 < kConsumerWarps; ++w8) u += tiles[(size_t)w8 * RP * RP + r * RP + q];
    t.Ups[(int64_t)2 * RR + e] = u;
    m2 = fma(u, __ldcg(t.Ups + e) * __ldcg(t.Ups + RR + e), m2);
  }
  consumer_sum3(m2, in, fl, sred);
  if (tid == 0) {
    const double f = 0.5 * t.normZ2[0] - in + 0.5 * m2;
    t.out[0] = f;
    t.out[1] = f - fl;
    t.out[2] = 0.0;
    t.out[3] = -1.0;
  }
#ifdef CP_TAIL_TIMING
  TAIL_T(6)
  if (tid == 0)
    printf("TAIL final cta %d: t0 %llu fence+bar %llu tick/flag %llu solve %llu gtick %llu dots+gram %llu reduce+out %llu\n",
           (int)blockIdx.x, tt[0], tt[1] - tt[0], tt[2] - tt[1], tt[3] - tt[2], tt[4] - tt[3], tt[5] - tt[4], tt[6] - tt[5]);
#endif
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

template <int NT, int MT, int OP, bool FEAT>
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
  // (PDL) predecessor's At / factor writes visible from here on; with p.prefetch the producer
  // warp first issues the Z part of its first stages and waits inside produce()
  const bool prefetch = FEAT && p.prefetch != 0 && p.Mout == nullptr;
  if (!(prefetch && (tid >> 5) == kConsumerWarps)) griddep();
  CTL_AFTER_WAIT
  // one-launch cp_mttkrp, mode 0: CTA 0 claims the grid barrier's words for this launch
  if (FEAT && OP == OP_MTTKRP && p.mode == 0 && p.Mout != nullptr && blockIdx.x == 0 && tid == 0) grid_claim(p.tick, p.tag);

  if (warp == kConsumerWarps) {
    produce<8, 2, FEAT>(p, lane, v0, v1, row0, Wb, sm, prefetch);  // (template args only select the TMA path)
    return;
  }
  if (warp == kConsumerWarps + 1) {
    // weight rows (returns at once when direct_w), then the optional Gamma job of CTA 0
    form_weights(p, lane, sm);
    if (p.gj.on && blockIdx.x == 0) {
      if (FEAT && p.gj.gram_rows > 0) gram_rows_warp<NT>(p.gj, lane);
      gamma_job_run(p.gj, sm.gjbuf, lane, 32, false);
    }
    if (FEAT && OP == OP_MTTKRP && p.tail.on && blockIdx.x == 0) {
      // publish the job's L^{-1}, Gram totals and status to the tail solves of every CTA
      __threadfence();
      __syncwarp();
      if (lane == 0) atomicExch(p.tail.gjflag, 1u);
    }
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
  const int bcs = P_FCM(p) ? 1 : wstride;
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
    boff[n] = (nok[n] ? n * 8 + gq : 0) * (P_FCM(p) ? p.fs : 1);
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
#ifdef CP_STREAM_TIMING
  long long tc_wait = 0, tc_n = 0, tc0 = clock64(), tc_flush = 0, tc_nflush = 0;
  unsigned long long tg0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tg0));
#endif
  for (;;) {
#ifdef CP_STREAM_TIMING
    const long long tcw = clock64();
#endif
    mbar_wait(p.direct_w ? &sm.full[stage] : &sm.wready[stage], fph);
#ifdef CP_STREAM_TIMING
    tc_wait += clock64() - tcw;
    ++tc_n;
#endif
#ifdef CP_CTA_TIMELINE
    if (tl_first == 0) tl_first = cta_gtimer();
#endif
    const int *h = sm.hdr + stage * kHdrInts;
    const int ncols = h[0];
    const int flags = h[1];
    const int slot = h[2];
    const double *zs = sm.zbuf + (size_t)stage * p.zst + arow0;
    const double *ws = (p.direct_w ? sm.abuf : sm.wbuf) + (size_t)stage * bstage + (P_FCM(p) ? h[3] : 0);
    // Khatri-Rao rows = staged factor rows x S, S = product of the slow digits' rows (staged by
    // the producer; S = 1 when there are none)
    double sl[NT];
#pragma unroll
    for (int n = 0; n < NT; ++n) sl[n] = 1.0;
    if (p.srows) {
#pragma unroll
      for (int j = 1; j < kMaxDigits; ++j) {
        if (j < p.nd && p.ord[j] != p.mode) {
          const double *sr = sm.sbuf + ((size_t)stage * kMaxDigits + j) * p.srs + gq * p.sstr + (P_FCM(p) ? (h[4 + j] & 1) : 0);
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
#ifdef CP_EXPERIMENTS
    if (p.dbg & 1) k0 = ncols;  // (CP_STREAM_DBG=1: consumers only hand the stages back -- the TMA ring alone)
#endif
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

#ifdef CP_STREAM_TIMING
    const long long tcf = clock64();
#endif
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
      const double *a1b = P_FCM(p) ? p.Af[0] + row0 : p.At[0] + row0 * p.RS;
      const int64_t a1rs = P_FCM(p) ? 1 : p.RS, a1cs = P_FCM(p) ? p.dims[0] : 1;
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
#ifdef CP_STREAM_TIMING
    if (flags & 1) {
      tc_flush += clock64() - tcf;
      ++tc_nflush;
    }
#endif
    if (flags & 2) break;
  }
#ifdef CP_CTA_TIMELINE
  tl_loop = cta_gtimer();
#endif
#ifdef CP_STREAM_TIMING
  // (timing build, tools/one_c4a_sweep.py: the consumers' share of the loop spent waiting for data)
#if CP_STREAM_TIMING >= 2  // (every CTA: the launch's distribution of loop times, tools/cta_loop_times.py)
  if (lane == 0 && warp == 0) {
#else
  if (lane == 0 && (warp == 0 || warp == 7) && (blockIdx.x == 0 || blockIdx.x == 101)) {
#endif
    unsigned long long tg1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tg1));
    const long long cyc = clock64() - tc0;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    printf("[cta %d warp %d op %d sm %u] consumer: loop %lld cycles in %llu ns (%.0f MHz) wait_full %lld stages %lld flush %lld in %lld segment ends start %llu\n", blockIdx.x,
           warp, OP, smid, cyc, tg1 - tg0, 1e3 * (double)cyc / (double)(tg1 - tg0), tc_wait, tc_n, tc_flush, tc_nflush, tg0);
  }
#endif
  if (FEAT && OP == OP_MTTKRP && p.mode != 0 && p.tail.on) sweep_tail<NT>(p, v0, v1, sm.zbuf);
  else if (FEAT && OP == OP_MTTKRP && p.mode != 0 && p.Mout != nullptr) mttkrp_complete_segments(p, v0, v1);

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
    if (FEAT && p.Mout != nullptr) {
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

template <int NT, int MT, int OP, bool FEAT>
cudaError_t launch_stream_mma_t(const StreamPlan &p, cudaStream_t st) {
  auto kern = stream_mma_kernel<NT, MT, OP, FEAT>;
  if (cudaError_t e = ensure_smem_attr((const void *)kern, 200 * 1024)) return e;
  return launch_kc(kPdlStream, kern, dim3(p.Gc * p.RB), dim3(kStreamThreads), (size_t)p.smem_bytes, st, p);
}

}  // namespace cpk
