// microbenchmark: cycles of the warp-register Cholesky + L^{-1} (copied from ylsolve.cu)
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
// 1/sqrt(x) for x > 0: the MUFU approximation (rsqrt.approx.f64) and two Newton steps in
// fp64 -- inline, no slow-path call (CUDA's rsqrt(double) calls a subroutine whose register
// save/restore dominated the factorization inside the solve kernels).
__device__ __forceinline__ double ys_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx, y * y, 1.5);
  y = y * fma(-hx, y * y, 1.5);
  return y;
}

// Cholesky Gamma = L L^T by one warp in shared memory (right-looking, no pivoting; a
// non-positive or NaN pivot sets *fail), then L^{-1} by forward substitution (lane c = column
// c); 1/L(j,j) = ys_rsqrt(pivot).  Every loop is rolled: this code runs once per block, and
// measured inside these kernels a fully unrolled register version was bound by instruction
// fetch (~7000 cycles per step against ~300 in isolation), so code size sets its latency.
template <int R>
__device__ __noinline__ void ys_chol_warp(double *sL, double *sLi, double *sDi, int *fail, int lane) {
  constexpr int LS = R + 1;
  bool ok = true;
#pragma unroll 1
  for (int j = 0; j < R; ++j) {
    const double piv = sL[j * LS + j];
    ok = ok && (piv > 0.0);
    const double inv = ys_rsqrt(ok ? piv : 1.0);
    __syncwarp();
    if (lane == j) {
      sL[j * LS + j] = piv * inv;
      sDi[j] = inv;
    } else if (lane > j && lane < R) {
      sL[lane * LS + j] *= inv;
    }
    __syncwarp();
    const int m = R - j - 1;
#pragma unroll 1
    for (int t = lane; t < m * m; t += 32) {
      const int ii = j + 1 + t / m, kk = j + 1 + t % m;
      if (kk <= ii) sL[ii * LS + kk] = fma(-sL[ii * LS + j], sL[kk * LS + j], sL[ii * LS + kk]);
    }
    __syncwarp();
  }
  if (!ok) {
    if (lane == 0) *fail = 1;
    return;
  }
  const int c = lane;
#pragma unroll 1
  for (int i = 0; i < R; ++i) {
    double s0 = (i == c) ? 1.0 : 0.0, s1 = 0.0;
    int k = c;
#pragma unroll 1
    for (; k + 1 < i; k += 2) {
      s0 = fma(-sL[i * LS + k], sLi[k * LS + c], s0);
      s1 = fma(-sL[i * LS + k + 1], sLi[(k + 1) * LS + c], s1);
    }
    if (k < i) s0 = fma(-sL[i * LS + k], sLi[k * LS + c], s0);
    if (c < R) sLi[i * LS + c] = (i >= c) ? (s0 + s1) * sDi[i] : 0.0;
  }
  __syncwarp();
}

template <int R>
__global__ void __cluster_dims__(8, 1, 1) kcholc(const double *G, double *out, long long *cyc, int variant) {
  constexpr int LS = R + 1;
  __shared__ double sL[R * LS], sLi[R * LS], sDi[R];
  __shared__ int fail;
  const int lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) sL[(e / R) * LS + e % R] = G[e];
  fail = 0;
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x < 32) ys_chol_warp<R>(sL, sLi, sDi, &fail, lane);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int R>
__global__ void kchol(const double *G, double *out, long long *cyc, int variant) {
  constexpr int LS = R + 1;
  __shared__ double sL[R * LS], sLi[R * LS], sDi[R];
  __shared__ int fail;
  const int lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) sL[(e / R) * LS + e % R] = G[e];
  fail = 0;
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x < 32) ys_chol_warp<R>(sL, sLi, sDi, &fail, lane);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) out[e] = sLi[(e / R) * LS + e % R];
}
int main() {
  const int R = 16;
  double G[R * R];
  for (int i = 0; i < R; ++i) for (int j = 0; j < R; ++j) G[i * R + j] = (i == j ? R + 1.0 : 0.5);
  double *dG, *dO; long long *dc;
  cudaMalloc(&dG, sizeof(G)); cudaMalloc(&dO, sizeof(G)); cudaMalloc(&dc, 8 * 256);
  cudaMemcpy(dG, G, sizeof(G), cudaMemcpyHostToDevice);
  for (int it = 0; it < 6; ++it) {
    cudaMemset(dO, 0, sizeof(G));
    const int nb = (it % 3 == 0) ? 1 : (it % 3 == 1 ? 32 : 128), nt = (it % 3 == 0) ? 32 : 256;
    kchol<R><<<nb, nt>>>(dG, dO, dc, 0);
    long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    double O[R * R]; cudaMemcpy(O, dO, sizeof(O), cudaMemcpyDeviceToHost);
    // check L^{-1} G L^{-T} = I via (L^{-1}) rows: max |(Li G Li^T) - I|
    double err = 0;
    for (int i = 0; i < R; ++i) for (int j = 0; j < R; ++j) { double t = 0; for (int a = 0; a < R; ++a) for (int b = 0; b < R; ++b) t += O[i*R+a]*G[a*R+b]*O[j*R+b]; err = fmax(err, fabs(t - (i==j))); }
    printf("chol R=%d blocks %d x %d: %lld cycles (block 0), err %.2e\n", R, nb, nt, c, err);
  }
  for (int it = 0; it < 2; ++it) {
    kcholc<R><<<128, 256>>>(dG, dO, dc, 0);
    long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("cluster kernel: chol %lld cycles (block 0) err %s\n", c, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
