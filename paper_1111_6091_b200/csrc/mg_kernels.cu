// mg_kernels.cu -- small device kernels used by the multigrid driver (mg_driver.cu) and exported
// through the C ABI: the normalization / ordering of the CP factors (eq:ALSnorm P:122-125,
// P:126) and a vector linear combination (FAS right-hand sides and corrections,
// eq:FASrhs P:342-345, eq:FASCGC P:347-349).
#include <cmath>

#include "mg_kernels.cuh"
#include "small_kernels.cuh"

namespace cpk {

// One block (256 threads).  lambda_r = (prod_n ||a_r^(n)||)^{1/N};
// a_r^(n) <- lambda_r a_r^(n) / ||a_r^(n)||  (components with a zero column are left as they are,
// lambda_r = 0); then the components are reordered by decreasing lambda (stable).
__global__ void __launch_bounds__(256) normalize_sort_kernel(const NormArgs a) {
  __shared__ double snrm[CP_MAX_N][CP_MAX_R];
  __shared__ double slam[CP_MAX_R];
  __shared__ int sperm[CP_MAX_R];
  __shared__ double sred[256];
  const int tid = threadIdx.x, R = a.R;
  for (int n = 0; n < a.N; ++n) {
    const int64_t I = a.dims[n];
    for (int r = 0; r < R; ++r) {
      double s = 0.0;
      for (int64_t i = tid; i < I; i += blockDim.x) {
        const double v = a.A[n][i + I * r];
        s = fma(v, v, s);
      }
      const double t = block_sum_256(s, sred);
      if (tid == 0) snrm[n][r] = sqrt(t);
    }
  }
  __syncthreads();
  if (tid == 0) {
    for (int r = 0; r < R; ++r) {
      double prod = 1.0;
      for (int n = 0; n < a.N; ++n) prod *= snrm[n][r];
      slam[r] = pow(prod, 1.0 / (double)a.N);
      sperm[r] = r;
    }
    if (a.sort) {
      for (int i = 1; i < R; ++i) {  // stable insertion sort, decreasing lambda
        const int v = sperm[i];
        int j = i - 1;
        while (j >= 0 && slam[sperm[j]] < slam[v]) {
          sperm[j + 1] = sperm[j];
          --j;
        }
        sperm[j + 1] = v;
      }
    }
  }
  __syncthreads();
  // scale into the temporary buffer in the new order, then copy back
  for (int n = 0; n < a.N; ++n) {
    const int64_t I = a.dims[n];
    for (int64_t e = tid; e < I * R; e += blockDim.x) {
      const int64_t i = e % I;
      const int r = (int)(e / I);
      const int src = sperm[r];
      const double nrm = snrm[n][src];
      double v = a.A[n][i + I * src];
      bool pos = true;
      for (int m = 0; m < a.N; ++m) pos = pos && (snrm[m][src] > 0.0);
      if (pos) v = slam[src] * (v / nrm);
      a.tmp[a.off[n] + e] = v;
    }
  }
  __syncthreads();
  for (int n = 0; n < a.N; ++n) {
    const int64_t I = a.dims[n];
    for (int64_t e = tid; e < I * R; e += blockDim.x) a.A[n][e] = a.tmp[a.off[n] + e];
  }
  if (a.lambda != nullptr && tid < R) a.lambda[tid] = slam[sperm[tid]];
}

// out = alpha * x + beta * y  (elementwise; out may alias x or y)
__global__ void lincomb_kernel(double *out, double alpha, const double *x, double beta,
                               const double *y, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = alpha * x[i] + (y != nullptr ? beta * y[i] : 0.0);
}

// one thread per output entry (row j, rank r) of every mode; dense rows of T are summed in
// ascending order
__global__ void __launch_bounds__(256) xfer_kernel(const XferArgs a) {
  griddep();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.off[a.N]) return;
  int n = 0;
  while (e >= a.off[n + 1]) ++n;
  const int64_t o = e - a.off[n];
  const int64_t ro = a.rows_out[n], ri = a.rows_in[n];
  const int64_t r = o / ro, j = o - r * ro;
  const double *x = a.x[n], *y = a.y[n];
  double v = 0.0;
  if (a.coarsen[n]) {
    const double *T = a.T[n] + j;
    const double *xc = x + ri * r, *yc = (y != nullptr) ? y + ri * r : nullptr;
    if (a.op == kXferApply) {
      for (int64_t i = 0; i < ri; ++i) v = fma(T[ro * i], xc[i], v);
    } else if (a.op == kXferFasRhs) {  // T (y - x), y optional
      for (int64_t i = 0; i < ri; ++i) v = fma(T[ro * i], (yc != nullptr ? yc[i] : 0.0) - xc[i], v);
    } else {                           // T (x - y)
      for (int64_t i = 0; i < ri; ++i) v = fma(T[ro * i], xc[i] - yc[i], v);
    }
  } else {
    const int64_t q = j + ri * r;
    if (a.op == kXferApply) v = x[q];
    else if (a.op == kXferFasRhs) v = (y != nullptr ? y[q] : 0.0) - x[q];
    else v = x[q] - y[q];
  }
  if (a.op == kXferApply) {
    a.dst[n][o] = v;
  } else if (a.op == kXferFasRhs) {
    a.dst[n][o] = a.z[n][o] + v;
    a.dst2[n][o] = a.w[n][o];
  } else {
    a.dst[n][o] += v;
  }
}

cudaError_t launch_xfer(XferArgs &a, cudaStream_t st) {
  a.off[0] = 0;
  for (int n = 0; n < a.N; ++n) a.off[n + 1] = a.off[n] + a.rows_out[n] * a.R;
  const int64_t tot = a.off[a.N];
  const unsigned blocks = (unsigned)((tot + 255) / 256);
  return launch_k(xfer_kernel, dim3(blocks > 0 ? blocks : 1), dim3(256), 0, st, a);
}

cudaError_t launch_normalize_sort(const NormArgs &a, cudaStream_t st) {
  normalize_sort_kernel<<<1, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_lincomb(double *out, double alpha, const double *x, double beta, const double *y,
                           int64_t n, cudaStream_t st) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 1024) blocks = 1024;
  if (blocks < 1) blocks = 1;
  lincomb_kernel<<<blocks, 256, 0, st>>>(out, alpha, x, beta, y, n);
  return cudaGetLastError();
}

}  // namespace cpk
