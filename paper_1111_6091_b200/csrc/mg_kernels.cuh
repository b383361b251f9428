// mg_kernels.cuh -- small device helpers of the multigrid driver (mg_kernels.cu).
#pragma once
#include "cp_internal.cuh"

namespace cpk {

struct NormArgs {
  int N, R, sort;
  int64_t dims[CP_MAX_N];
  int64_t off[CP_MAX_N];  // offsets of the factors in tmp
  double *A[CP_MAX_N];
  double *tmp;     // sum_n I_n * R doubles
  double *lambda;  // R (device) or null
};

// Fused transfer operations of one multigrid level, all N modes in ONE launch (the FAS cycle of
// Algorithm 2 issued ~8N tiny launches per level pair: mode products of the I x R factor
// matrices, vector combinations and copies).  Per mode n the operator T[n] is dense, column-major
// (rows_out x rows_in), or the identity when coarsen[n] == 0 (rows_out == rows_in):
//   kXferApply  : dst = T x                                     (restriction R A, interpolation Phat A_c)
//   kXferFasRhs : dst = z + T (y - x)  [y may be null: 0],  dst2 = w   (F_c = H_c(A~_c) + R (F - H(A)),
//                 A_c = A~_c; eq:FASrhs)
//   kXferCorrect: dst = dst + T (x - y)                         (A += Phat (A_c - A~_c); eq:FASCGC)
// x, y, z, w: rows_in x R (z, w, dst2: rows_out x R for kXferFasRhs), column-major.
enum { kXferApply = 0, kXferFasRhs = 1, kXferCorrect = 2 };
struct XferArgs {
  int N, R, op;
  int64_t rows_in[CP_MAX_N], rows_out[CP_MAX_N];
  int coarsen[CP_MAX_N];
  const double *T[CP_MAX_N];
  const double *x[CP_MAX_N], *y[CP_MAX_N], *z[CP_MAX_N], *w[CP_MAX_N];
  double *dst[CP_MAX_N], *dst2[CP_MAX_N];
  int64_t off[CP_MAX_N + 1];  // prefix sums of the output entries rows_out * R
};
cudaError_t launch_xfer(XferArgs &a, cudaStream_t st);

cudaError_t launch_normalize_sort(const NormArgs &a, cudaStream_t st);
cudaError_t launch_lincomb(double *out, double alpha, const double *x, double beta, const double *y,
                           int64_t n, cudaStream_t st);

}  // namespace cpk
