// probe_read_pattern.cu -- HBM read bandwidth of 1 GiB against the CTA-to-address assignment:
//   0: grid-stride tiles (all CTAs read one compact window that moves through the tensor: norm2's pattern)
//   1: one contiguous range per CTA (the streaming kernels' v-ranges: G streams P/G apart)
//   2: contiguous ranges per CTA *pair* (two CTAs alternate tiles of one range)
//   3: grid-stride over super-tiles of S tiles (each CTA reads S consecutive tiles, then jumps by G S)
// 296 CTAs x 256 threads, 32 KB tiles, 8 independent 16-byte loads per thread per tile.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 2) rd(const double2 *z, long ntiles, int mode, int S, double *out) {
  const long G = gridDim.x, b = blockIdx.x;
  double acc = 0.0;
  auto tile = [&](long t) {
    const double2 *p = z + t * 2048 + threadIdx.x;
    double2 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcs(p + j * 256);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j].x + v[j].y;
  };
  if (mode == 0) {
    for (long t = b; t < ntiles; t += G) tile(t);
  } else if (mode == 1) {
    const long t0 = ntiles * b / G, t1 = ntiles * (b + 1) / G;
    for (long t = t0; t < t1; ++t) tile(t);
  } else if (mode == 2) {
    const long pr = b >> 1, P2 = G >> 1;
    const long t0 = ntiles * pr / P2, t1 = ntiles * (pr + 1) / P2;
    for (long t = t0 + (b & 1); t < t1; t += 2) tile(t);
  } else {
    const long nsuper = ntiles / S;
    for (long s = b; s < nsuper; s += G)
      for (int k = 0; k < S; ++k) tile(s * S + k);
  }
  if (acc == 123.456) out[0] = acc;
}

int main() {
  const long bytes = 1L << 30, ntiles = bytes / 32768;
  double2 *z; double *out;
  cudaMalloc(&z, bytes); cudaMalloc(&out, 8); cudaMemset(z, 0, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](int mode, int S, const char *label) {
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0); rd<<<296, 256>>>(z, ntiles, mode, S, out); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    printf("%-46s %.1f us  %.0f GB/s\n", label, best * 1e3, bytes / best / 1e6);
  };
  run(0, 1, "grid-stride tiles (compact window)");
  run(1, 1, "contiguous range per CTA (296 streams)");
  run(2, 1, "contiguous range per CTA pair (148 streams)");
  run(3, 4, "grid-stride super-tiles of 4 (128 KB)");
  run(3, 16, "grid-stride super-tiles of 16 (512 KB)");
  run(3, 64, "grid-stride super-tiles of 64 (2 MB)");
  run(0, 1, "grid-stride tiles again");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
