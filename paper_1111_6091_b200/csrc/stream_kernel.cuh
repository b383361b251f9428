// stream_kernel.cuh -- the Z-streaming kernel of libcp.so: MTTKRP (eq:gradEqn, eq:Phi,
// P:104-111) and the residual pass of cp_fit (eq:CPfunctional).
//
// Design:
//  * Z is viewed as an I1 x Q column-major matrix (mode-1 fibers are columns).  Every mode's
//    MTTKRP streams Z in that order: a thread owns fixed rows i1 (2 per thread) for the whole
//    pass and keeps R accumulators per row in registers, so the Khatri-Rao row w_q of a column
//    is formed ONCE per column (by the producer warp, into shared memory) and broadcast to all
//    rows of the column -- the "reuse along the fast mode" of the north star.
//  * One producer warp feeds a ring of shared-memory stages with TMA bulk copies
//    (cp.async.bulk + mbarrier complete_tx); 8 consumer warps do R DFMAs per element.
//  * mode 0 (paper mode 1): the output rows are the owned rows; each column group writes
//    an I1 x R partial, reduced in fixed order by the next kernel (no atomics).
//  * mode m >= 1: columns are visited with i_m outermost; at the end of each i_m segment the
//    consumers contract their accumulators with A^(1) rows and reduce across the CTA
//    (warp shuffles + shared memory), writing one R-vector partial per (CTA, segment).
#pragma once
#include "cp_internal.cuh"

namespace cpk {

// v-order odometer: digit j has radix p.rad[j] and is the index of mode p.ord[j]
// (fastest first).  add_carry adds a small non-negative c; digits_to_q maps to the column q.
__device__ __forceinline__ void add_carry(int (&d)[kMaxDigits], int nd, const int *rad, int c) {
#pragma unroll
  for (int j = 0; j < kMaxDigits; ++j) {
    if (j < nd && c != 0) {
      const int t = d[j] + c;
      c = t / rad[j];
      d[j] = t - c * rad[j];
    }
  }
}
__device__ __forceinline__ int64_t digits_to_q(const StreamPlan &p, const int (&d)[kMaxDigits]) {
  int64_t q = 0;
#pragma unroll
  for (int j = 0; j < kMaxDigits; ++j)
    if (j < p.nd) q += (int64_t)d[j] * p.qsd[j];
  return q;
}

template <int R, int V, int OP>
__global__ void __launch_bounds__(kStreamThreads, (R <= 16 ? 2 : 1)) stream_kernel(const __grid_constant__ StreamPlan p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int WSTR = (R % 2 == 0) ? R + 2 : R + 1;  // weight row stride (even: 16-B aligned)
  const int zst = p.cps * p.Wmax;                      // doubles per Z stage
  const int wst = p.cps * WSTR;                        // doubles per weight stage
  double *zbuf = reinterpret_cast<double *>(smem_raw);
  double *wbuf = zbuf + (size_t)p.nstages * zst;
  double *red = wbuf + (size_t)p.nstages * wst;        // [8][R] (+8 spare)
  uint64_t *full = reinterpret_cast<uint64_t *>(red + kConsumerWarps * R + 8);
  uint64_t *empty = full + p.nstages;
  int *hdr = reinterpret_cast<int *>(empty + p.nstages);  // [nstages][4]

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
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ============================ producer warp ============================
    // Columns are visited in "v order"; the producer keeps the v-digits of the
    // stage start in registers (an odometer over p.rad, 32-bit), so no 64-bit division runs
    // per column.  Lane 0 issues the TMA bulk copies; all lanes form the Khatri-Rao rows.
    const int cpp = 32 / R;  // weight columns per pass (lanes over (col, r))
    const int lc = lane / R, lr = lane - (lane / R) * R;
    const int nd = p.nd;
    int B[kMaxDigits];
    {
      int64_t t = v0;
#pragma unroll
      for (int j = 0; j < kMaxDigits; ++j) {
        B[j] = 0;
        if (j < nd) {
          B[j] = (int)(t % p.rad[j]);
          t /= p.rad[j];
        }
      }
    }
    int64_t seg_left = p.Qn - (v0 % p.Qn);
    int seg_slot = 0;
    int stage = 0;
    uint32_t eph = 1;
    int64_t v = v0;
    while (v < v1) {
      const int64_t lim = (seg_left < v1 - v) ? seg_left : (v1 - v);
      const int ncols = (int)(lim < p.cps ? lim : p.cps);
      const bool last = (v + ncols == v1);
      const bool eos = (ncols == seg_left) || last;  // a segment ends, or this CTA's range does
      mbar_wait(&empty[stage], eph);
      double *zs = zbuf + (size_t)stage * zst;
      if (V == 2) {
        if (lane == 0) {
          mbar_expect_tx(&full[stage], (uint32_t)(ncols * Wb * 8));
          int D[kMaxDigits];
#pragma unroll
          for (int j = 0; j < kMaxDigits; ++j) D[j] = B[j];
          int64_t q = digits_to_q(p, D);
          int64_t run_q = q;
          int run_col = 0, run_n = 1;
          for (int col = 1; col <= ncols; ++col) {
            int64_t q2 = -1;
            if (col < ncols) {
              add_carry(D, nd, p.rad, 1);
              q2 = digits_to_q(p, D);
            }
            if (col < ncols && p.RB == 1 && q2 == q + 1) {
              ++run_n;
            } else {
              bulk_g2s(zs + (size_t)run_col * Wb, p.Z + run_q * p.I1 + row0, (uint32_t)(run_n * Wb * 8),
                       &full[stage]);
              run_q = q2;
              run_col = col;
              run_n = 1;
            }
            q = q2;
          }
        }
      } else {
        // scalar fallback (odd I1: columns are not 16-B aligned): the warp copies elements
        int D[kMaxDigits];
#pragma unroll
        for (int j = 0; j < kMaxDigits; ++j) D[j] = B[j];
        for (int col = 0; col < ncols; ++col) {
          if (col > 0) add_carry(D, nd, p.rad, 1);
          const double *src = p.Z + digits_to_q(p, D) * p.I1 + row0;
          for (int i = lane; i < Wb; i += 32) zs[(size_t)col * Wb + i] = __ldg(src + i);
        }
      }
      // Khatri-Rao rows w_q[r] = prod_{k>=1, k != mode} A^(k)(i_k, r) of this stage's columns,
      // four columns per lane at a time so their factor loads are in flight together
      double *ws = wbuf + (size_t)stage * wst;
      if (lc < cpp) {
        for (int c0 = lc; c0 < ncols; c0 += 4 * cpp) {
          int D[4][kMaxDigits];
          double w[4];
#pragma unroll
          for (int u4 = 0; u4 < 4; ++u4) {
#pragma unroll
            for (int j = 0; j < kMaxDigits; ++j) D[u4][j] = B[j];
            add_carry(D[u4], nd, p.rad, c0 + u4 * cpp);
            w[u4] = 1.0;
          }
#pragma unroll
          for (int j = 0; j < kMaxDigits; ++j) {
            if (j < nd && p.ord[j] != p.mode) {
              const double *a = p.At[p.ord[j]] + lr;
#pragma unroll
              for (int u4 = 0; u4 < 4; ++u4) w[u4] *= __ldg(a + D[u4][j] * R);
            }
          }
#pragma unroll
          for (int u4 = 0; u4 < 4; ++u4) {
            const int col = c0 + u4 * cpp;
            if (col < ncols) ws[col * WSTR + lr] = w[u4];
          }
        }
      }
      if (lane == 0) {
        int *h = hdr + stage * 4;
        h[0] = ncols;
        h[1] = (eos ? 1 : 0) | (last ? 2 : 0);
        h[2] = seg_slot;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[stage]);
      v += ncols;
      add_carry(B, nd, p.rad, ncols);
      seg_left -= ncols;
      if (seg_left == 0) {
        seg_left = p.Qn;
        ++seg_slot;
      }
      if (++stage == p.nstages) {
        stage = 0;
        eph ^= 1u;
      }
    }
    return;
  }

  // ============================ consumer warps ============================
  const int U = Wb / V;                       // row units per column in this block
  const int cpt = (kConsumers / U) > 0 ? (kConsumers / U) : 1;  // columns per sub-tile
  const int u = tid % U;
  const int sl = tid / U;
  const bool active = sl < cpt;

  double acc[V][R];
#pragma unroll
  for (int v = 0; v < V; ++v)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[v][r] = 0.0;

  double arow[OP == OP_RESID ? V : 1][OP == OP_RESID ? R : 1];
  if (OP == OP_RESID) {
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int r = 0; r < R; ++r)
        arow[v][r] = active ? __ldg(p.At[0] + (row0 + u * V + v) * R + r) : 0.0;
  }

  int stage = 0;
  uint32_t fph = 0;
  for (;;) {
    mbar_wait(&full[stage], fph);
    const int *h = hdr + stage * 4;
    const int ncols = h[0];
    const int flags = h[1];
    const int slot = h[2];
    const double *zs = zbuf + (size_t)stage * zst;
    const double *wsb = wbuf + (size_t)stage * wst;
    if (active) {
      for (int col = sl; col < ncols; col += cpt) {
        double z[V];
        if (V == 2) {
          const double2 zz = *reinterpret_cast<const double2 *>(zs + (size_t)col * Wb + 2 * u);
          z[0] = zz.x;
          z[V - 1] = zz.y;
        } else {
          z[0] = zs[(size_t)col * Wb + u];
        }
        const double *w = wsb + col * WSTR;
        if (OP == OP_MTTKRP) {
#pragma unroll
          for (int r = 0; r + 1 < R; r += 2) {
            const double2 ww = *reinterpret_cast<const double2 *>(w + r);
#pragma unroll
            for (int v = 0; v < V; ++v) {
              acc[v][r] = fma(z[v], ww.x, acc[v][r]);
              acc[v][r + 1] = fma(z[v], ww.y, acc[v][r + 1]);
            }
          }
          if (R & 1) {
            const double wl = w[R - 1];
#pragma unroll
            for (int v = 0; v < V; ++v) acc[v][R - 1] = fma(z[v], wl, acc[v][R - 1]);
          }
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
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == p.nstages) {
      stage = 0;
      fph ^= 1u;
    }

    if (OP == OP_MTTKRP && p.mode != 0 && (flags & 1)) {
      // ---- end of an i_m segment: contract with A^(1) rows and reduce over the CTA ----
      double pr[R];
#pragma unroll
      for (int r = 0; r < R; ++r) pr[r] = 0.0;
      if (active) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const double *a1 = p.At[0] + (row0 + u * V + v) * R;
#pragma unroll
          for (int r = 0; r < R; ++r) pr[r] = fma(__ldg(a1 + r), acc[v][r], pr[r]);
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int r = 0; r < R; ++r) acc[v][r] = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) pr[r] += __shfl_xor_sync(0xffffffffu, pr[r], off);
      }
      if (lane == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) red[warp * R + r] = pr[r];
      }
      named_bar_sync(1, kConsumers);
      if (tid < R) {
        double sum = 0.0;
#pragma unroll
        for (int w8 = 0; w8 < kConsumerWarps; ++w8) sum += red[w8 * R + tid];
        p.part[((int64_t)blockIdx.x * p.slots + slot) * R + tid] = sum;
      }
      named_bar_sync(1, kConsumers);
    }
    if (flags & 2) break;
  }

  if (OP == OP_MTTKRP && p.mode == 0) {
    // ---- mode 0: write this CTA's I1 x R partial for its row block (slots summed in order) ----
    double *out = p.part + (int64_t)c * p.I1 * R;
    if (cpt > 1) {
      named_bar_sync(1, kConsumers);  // every consumer is past the ring: reuse it
      double *sred = zbuf;            // Wb x R
      for (int s = 1; s < cpt; ++s) {
        if (active && sl == s) {
#pragma unroll
          for (int v = 0; v < V; ++v)
#pragma unroll
            for (int r = 0; r < R; ++r) sred[(u * V + v) + Wb * r] = acc[v][r];
        }
        named_bar_sync(1, kConsumers);
        if (sl == 0) {
#pragma unroll
          for (int v = 0; v < V; ++v)
#pragma unroll
            for (int r = 0; r < R; ++r) acc[v][r] += sred[(u * V + v) + Wb * r];
        }
        named_bar_sync(1, kConsumers);
      }
    }
    if (sl == 0) {
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int r = 0; r < R; ++r) out[row0 + u * V + v + p.I1 * r] = acc[v][r];
    }
  } else if (OP == OP_RESID) {
    double sacc = 0.0;
#pragma unroll
    for (int v = 0; v < V; ++v) sacc += acc[v][0];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, off);
    if (lane == 0) red[warp] = sacc;
    named_bar_sync(1, kConsumers);
    if (tid == 0) {
      double sum = 0.0;
      for (int w8 = 0; w8 < kConsumerWarps; ++w8) sum += red[w8];
      p.part[blockIdx.x] = sum;
    }
  }
}

template <int R, int V, int OP>
cudaError_t launch_stream_t(const StreamPlan &p, cudaStream_t st) {
  auto kern = stream_kernel<R, V, OP>;
  static bool attr_done = false;  // per instantiation
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  kern<<<p.Gc * p.RB, kStreamThreads, p.smem_bytes, st>>>(p);
  return cudaGetLastError();
}

using StreamLauncher = cudaError_t (*)(const StreamPlan &, cudaStream_t);

}  // namespace cpk
