// small_kernels.cuh -- argument structs of the R x R / reduction kernels (small_kernels.cu).
#pragma once
#include <cstring>

#include "cp_internal.cuh"
#include "gamma_job.cuh"

namespace cpk {

// ---------------------------------------------------------------- block reduction (fixed tree)
// blockDim.x == 256; returns the sum to every thread (warp xor trees, then the 8 warp sums in a
// fixed order; two barriers).
__device__ __forceinline__ double block_sum_256(double v, double *sred) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();  // (sred may still be read by a previous call)
  if (lane == 0) sred[w] = v;
  __syncthreads();
  return ((sred[0] + sred[1]) + (sred[2] + sred[3])) + ((sred[4] + sred[5]) + (sred[6] + sred[7]));
}
// three sums at once (sred: 24 doubles)
__device__ __forceinline__ void block_sum3_256(double &a, double &b, double &c, double *sred) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, off);
    b += __shfl_xor_sync(0xffffffffu, b, off);
    c += __shfl_xor_sync(0xffffffffu, c, off);
  }
  __syncthreads();
  if (lane == 0) {
    sred[w] = a;
    sred[8 + w] = b;
    sred[16 + w] = c;
  }
  __syncthreads();
  a = ((sred[0] + sred[1]) + (sred[2] + sred[3])) + ((sred[4] + sred[5]) + (sred[6] + sred[7]));
  b = ((sred[8] + sred[9]) + (sred[10] + sred[11])) + ((sred[12] + sred[13]) + (sred[14] + sred[15]));
  c = ((sred[16] + sred[17]) + (sred[18] + sred[19])) + ((sred[20] + sred[21]) + (sred[22] + sred[23]));
}

// Where the stream kernel left its partials, and how to sum them (fixed order).
struct ReduceGeom {
  int R, Gc, RB, slots, mode0;  // mode0: partials are I1 x R per column group
  int direct;                   // 1: part is M itself (In_rows x R, column-major)
  int64_t I1, Q, Qn, In;
  int64_t In_rows;  // rows of the output (I_mode)
  const double *part;
};

inline ReduceGeom reduce_geom(const StreamPlan &p) {
  ReduceGeom g;
  g.R = p.R;
  g.Gc = p.Gc;
  g.RB = p.RB;
  g.slots = p.slots;
  g.mode0 = (p.mode == 0) ? 1 : 0;
  g.direct = 0;
  g.I1 = p.I1;
  g.Q = p.Q;
  g.Qn = p.Qn;
  g.In = p.In;
  g.In_rows = (p.mode == 0) ? p.I1 : p.dims[p.mode];
  g.part = p.part;
  return g;
}

// Row blocking of the kernels that consume stream partials: sp threads per M entry (mode 0
// has Gc partials per entry), rpc rows per 256-thread CTA.
inline void row_blocking(const StreamPlan &p, int *rpc, int *sp) {
  int s = 1;
  if (p.mode == 0) {
    s = p.Gc / 16;
    if (s < 1) s = 1;
    if (s > 8) s = 8;
    while (s > 1 && p.R * s > 256) --s;
  }
  int r = 256 / (p.R * s);
  if (r < 1) r = 1;
  *sp = s;
  *rpc = r;
}

constexpr int kPrepRows = 64;  // rows per prep block

struct PrepArgs {
  int N, R;
  int blk_off[CP_MAX_N + 1];  // first block of mode k (blk_off[N] = grid size)
  int64_t dims[CP_MAX_N];
  const double *A[CP_MAX_N];
  double *At[CP_MAX_N];
  double *gpre;    // per-block partial Grams (may be null: no Grams)
  double *status;  // may be null
  int keep_status; // 1: leave status[0..1] as they are (a later sweep of one cp_als_sweeps call:
                   // an earlier failure stays reported and the later solves skip); tickets reset
  unsigned *zero;  // zeroed by block 0 (Y_L segment tickets), may be null
  int nzero;
};

// Where the prep kernel left the partial Grams of the input factors.
struct PrepGrams {
  const double *gpre;
  int blk_off[CP_MAX_N + 1];
  int nblk[CP_MAX_N];
  const double *tot;  // non-null: the Gram TOTALS (N x R x R) of the current factors instead of the
                      // prep partials -- a steady-state sweep (cp_als_sweeps, sweep k >= 1: the
                      // previous sweep left At and every Upsilon total current; no prep launch)
};

struct FinalizeArgs {
  int N, R, nlast, dot_stride;
  int nsolve[CP_MAX_N];
  const double *glast, *dotM_last, *dotF;
  double *Ups;
  const double *normZ2;
  double *status, *out;
};

// status area (8 doubles): [0] status, [1] failed mode, [kTicketSlot] completion ticket (u32)
constexpr int kTicketSlot = 4;
constexpr int kTicketSlot2 = 5;  // ylsolve: last-cluster ticket (zeroed by prep)

struct SolveArgs {
  int N, R, mode, prev_mode, nprev, rpc, sp;
  int64_t In;
  ReduceGeom rg;
  PrepGrams pg;
  const double *F;      // F^(mode) or null
  double *A;            // A^(mode), column-major (output)
  double *At;           // row-major copy (output)
  double *Ups;          // N x R x R Gram totals
  const double *gprev;  // previous mode's per-CTA partial Grams (null for mode 0)
  double *gcur;         // this kernel's per-CTA partial Grams
  double *dotM, *dotF;  // per-CTA <M,A>, <F,A>
  double *status;       // [0] status, [1] failed mode
  int fin_on;           // last solve of the sweep: the last block to finish runs the finalize
  int dbg;              // experiments only (CP_SOLVE_DBG): 1 = skip Gamma / Cholesky (L = I)
  const double *linv;   // L^{-1} of Gamma^(mode) from a Gamma job (gamma_job.cuh), or null:
                        // the solve forms Gamma and factors it itself
  unsigned *ticket;
  FinalizeArgs fin;
};

struct GradArgs {
  int N, R, mode, rpc, sp;
  int64_t In;
  ReduceGeom rg;
  PrepGrams pg;
  const double *A, *F, *Ups;
  double *G, *gpart;
  double *dpart;  // cp_gradient, last mode: per-CTA <M^(n), A^(n)> (f by expansion), or null
};

struct FitFinalArgs {
  int N, nresid, gstride;
  int ngrad[CP_MAX_N];
  const double *resid, *gpart, *normZ2;
  double *out;
  // cp_gradient (expand = 1): f = 1/2 ||Z||^2 - <M^(N), A^(N)> + 1/2 1^T (*_k Upsilon^(k)) 1
  // from the last mode's <M, A> partials and the prep Grams, instead of the residual pass
  int expand, R, ndot;
  const double *dpart;
  PrepGrams pg;
};

__global__ void reduce_mttkrp_kernel(const ReduceGeom g, int rpc, int sp, double *M);
__global__ void reduce_mode0_kernel(const double *part, int Gc, int64_t S, double *M);
__global__ void finalize_sweep_kernel(const FinalizeArgs a);
__global__ void gradient_kernel(const GradArgs a);
__global__ void finalize_fit_kernel(const FitFinalArgs a);
__global__ void norm2_kernel(const double *__restrict__ Z, int64_t P, double *part);
__global__ void norm2_final_kernel(const double *part, int n, double *out);
cudaError_t launch_solve(const SolveArgs &a, int grid, cudaStream_t st);

// ---- dimension-tree sweep (NEXT-4): Y_L(i0, i1, r) = sum_{i_2..} z * prod_{k>=2} A^(k)(i_k, r)
// written by the OP_YL stream pass (full segments in yl, shared ones in per-CTA edge blocks)
struct YLGeom {
  int R, Gc, RB, Wmax;
  int64_t I0, I1, Q, Qn;
  const double *yl, *edge;
};
inline ReduceGeom direct_geom(const double *M, int64_t rows, int R) {
  ReduceGeom g;
  memset(&g, 0, sizeof(g));
  g.R = R;
  g.direct = 1;
  g.In_rows = rows;
  g.part = M;
  return g;
}
// completes the segments split between CTAs (edge blocks -> yl)
cudaError_t launch_yl_fixup(const YLGeom &y, cudaStream_t st);
// partials of M0(i0, r) = sum_{i1} Y_L(i0, i1, r) A^(1)(i1, r) (A1: column-major I1 x R):
// part[b][r][i0] for b < ymm0_ranges(y) -- summed in b order by the mode-0 solve
int ymm0_ranges(int R, int64_t I1);
// row blocking (rows per CTA, threads per entry) of the mode-0 solve that sums those partials
void ymm0_solve_blocking(int R, int64_t I1, int *rpc, int *sp);
cudaError_t launch_ymm0(const YLGeom &y, const double *A1, double *part, cudaStream_t st);
// M1(i1, r) = sum_{i0} Y_L(i0, i1, r) A^(0)(i0, r)   (A0: column-major I0 x R)
cudaError_t launch_ymm1(const YLGeom &y, const double *A0, double *M1, const GammaJob &gj, cudaStream_t st);
// M_m(i_m, r) = sum_{j: i_m(j)} Y_R(j, r) prod_{k >= 2, k != m} A^(k)(i_k(j), r), j over modes 2..N-1
struct YRArgs {
  int N, R, RS, mode;
  GammaJob gj;  // optional: run by one extra block
  int64_t dims[CP_MAX_N];
  const double *At[CP_MAX_N];
  const double *YR;  // J x R column-major, J = prod_{k >= 2} I_k (mode 2 fastest)
  double *M;
};
cudaError_t launch_yr(const YRArgs &a, cudaStream_t st);

// ylsolve.cu: mode 0 / mode 1 of the dimension-tree sweep -- M rows from Y_L, Gamma, Cholesky
// and the row solves in one kernel (blocks of 4 rows, 8-CTA clusters).
struct YLSolveArgs {
  int N, R, mode;          // mode 0 or 1
  int RS;                  // mode 0: row stride of Bfac (At^(1)); unused for mode 1
  int RSo;                 // row stride of the At output
  int64_t I0, I1, In;      // Y_L dims; rows of this mode
  const double *yl;        // Y_L [i1][r][i0]
  const double *Bfac;      // mode 0: At^(1) (row-major, previous sweep); mode 1: A^(0)_new (column-major)
  PrepGrams pg;            // Grams of the factors not updated yet (prep partials)
  const double *gin;       // mode 1: per-cluster partial Grams of A^(0)_new
  int nin;
  const double *linv;      // optional L^{-1} of Gamma^(mode) from a Gamma job (else factored in-block)
  int ups_total;           // bit k: Upsilon^(k) is read as the total Ups[k] (else summed from partials)
  double *total;           // optional: the last cluster writes the Gram total of the new factor here
  unsigned *ticket;        // (zero; reset by the last cluster)
  const double *F;         // F^(mode) or null
  double *A, *At;          // outputs: column-major factor, row-major copy
  double *Ups;             // Gram totals (block 0 writes the ones it sums)
  double *gcur;            // per-cluster partial Grams of the new rows
  double *dotF;            // per-cluster <F, A>
  double *status;
  int vec1;                // mode 1: Y_L rows and A^(0)_new columns read as 32-byte vectors (I0 % 4 == 0,
                           // 32-B aligned A^(0)_new)
};
int ylsolve_clusters(int64_t In);  // grid = 8 x this
cudaError_t launch_ylsolve(const YLSolveArgs &a, cudaStream_t st);
cudaError_t launch_prep(const PrepArgs &a, cudaStream_t st);

// Fill the prep block offsets for a shape (blocks of kPrepRows rows per mode).
inline void prep_blocks(const cp_shape &s, PrepArgs &pa, PrepGrams &pg) {
  int off = 0;
  for (int k = 0; k < s.N; ++k) {
    const int nb = (int)((s.dims[k] + kPrepRows - 1) / kPrepRows);
    pa.blk_off[k] = pg.blk_off[k] = off;
    pg.nblk[k] = nb;
    off += nb;
  }
  pa.blk_off[s.N] = pg.blk_off[s.N] = off;
}

}  // namespace cpk
