// probe_clock.cu -- SM clock (clock64 / globaltimer) inside a pure streaming-read kernel, for comparison
// with the clocks the timing build of the streaming kernels prints.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 2) rd(const double2 *z, long ntiles, double *out) {
  unsigned long long g0, g1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  const long long c0 = clock64();
  double acc = 0.0;
  for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const double2 *p = z + t * 2048 + threadIdx.x; double2 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcs(p + j * 256);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j].x + v[j].y;
  }
  const long long c1 = clock64(); asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == 101)) printf("[cta %d] read loop %lld cycles in %llu ns (%.0f MHz)\n", blockIdx.x, c1 - c0, g1 - g0, 1e3 * (double)(c1 - c0) / (double)(g1 - g0));
  if (acc == 123.456) out[0] = acc;
}
int main() {
  const long bytes = 1L << 30; double2 *z; double *out; cudaMalloc(&z, bytes); cudaMalloc(&out, 8); cudaMemset(z, 0, bytes);
  for (int r = 0; r < 3; ++r) { rd<<<296, 256>>>(z, bytes / 32768, out); cudaDeviceSynchronize(); }
  return 0;
}
