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

cudaError_t launch_normalize_sort(const NormArgs &a, cudaStream_t st);
cudaError_t launch_lincomb(double *out, double alpha, const double *x, double beta, const double *y,
                           int64_t n, cudaStream_t st);

}  // namespace cpk
