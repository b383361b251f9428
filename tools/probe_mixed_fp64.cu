// probe_mixed_fp64.cu -- are DFMA and DMMA (mma.sync m8n8k4 f64) separate pipes on sm_100a?
// Times a DFMA-only kernel, a DMMA-only kernel and mixes (warp-split and per-warp interleaved) with
// the same per-kernel work; if the mixed kernels take ~max(t_f, t_m) the pipes are separate, if
// ~t_f + t_m they share the FP64 units.   nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma8(double (&d)[8][2], double a, double b) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dfma8(double (&acc)[8], double a, double b) {
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], a, b);
}

// mode 0: all warps DFMA (nf iterations); 1: all warps DMMA (nm iterations);
// 2: even warps DMMA nm, odd warps DFMA nf; 3: every warp interleaves nm DMMA groups with nf DFMA groups
__global__ void k(double *out, int mode, int nf, int nm, double a, double b) {
  double acc[8], d[8][2];
#pragma unroll
  for (int c = 0; c < 8; ++c) { acc[c] = threadIdx.x * 1e-3 + c; d[c][0] = c; d[c][1] = c + 1; }
  const int w = threadIdx.x >> 5;
  if (mode == 0) { for (int i = 0; i < nf; ++i) dfma8(acc, a, b); }
  else if (mode == 1) { for (int i = 0; i < nm; ++i) dmma8(d, a, b); }
  else if (mode == 2) {
    if (w & 1) { for (int i = 0; i < nf; ++i) dfma8(acc, a, b); }
    else { for (int i = 0; i < nm; ++i) dmma8(d, a, b); }
  } else {
    const int n = nf > nm ? nf : nm;
    for (int i = 0; i < n; ++i) { if (i < nm) dmma8(d, a, b); if (i < nf) dfma8(acc, a, b); }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c] + d[c][0] + d[c][1];
  if (s == 123.456) out[0] = s;
}

static float run(double *out, int mode, int nf, int nm, int blocks) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); k<<<blocks, 256>>>(out, mode, nf, nm, 1.0000001, 1e-9); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out; cudaMalloc(&out, 8);
  const int blocks = sms * 8, N = 20000;
  k<<<blocks, 256>>>(out, 0, 10, 10, 1.0, 1.0); cudaDeviceSynchronize();
  const double warps = 8.0 * blocks;
  const double fl_f = 2.0 * 8 * 32, fl_m = 2.0 * 8 * 8 * 4 * 8;   // per warp-iteration
  float tf = run(out, 0, N, 0, blocks), tm = run(out, 1, 0, N, blocks);
  printf("DFMA only: %.3f ms %.1f TFLOP/s\nDMMA only: %.3f ms %.1f TFLOP/s\n", tf, fl_f * N * warps / tf / 1e9, tm, fl_m * N * warps / tm / 1e9);
  // warp split: half the warps each, 2N iterations -> same total work as (DFMA only) + (DMMA only)
  float t2 = run(out, 2, 2 * N, 2 * N, blocks);
  printf("warp-split (same total work as both): %.3f ms  [sum %.3f, max %.3f]  combined %.1f TFLOP/s\n", t2, tf + tm, tf > tm ? tf : tm,
         (fl_f + fl_m) * N * warps / t2 / 1e9);
  float t3 = run(out, 3, N, N, blocks);
  printf("interleaved  (same total work as both): %.3f ms  [sum %.3f, max %.3f]  combined %.1f TFLOP/s\n", t3, tf + tm, tf > tm ? tf : tm,
         (fl_f + fl_m) * N * warps / t3 / 1e9);
  // DMMA-heavy mixes: DFMA share s of the flops
  for (int pct = 10; pct <= 50; pct += 10) {
    // per warp: nm DMMA groups (2048 fl each) + nf DFMA groups (512 fl each)
    int nm = N, nf = (int)((double)N * 4.0 * pct / (100 - pct));
    float t = run(out, 3, nf, nm, blocks);
    printf("interleaved DFMA share %d%% of flops: %.3f ms, %.1f TFLOP/s\n", pct, t, (fl_f * nf + fl_m * nm) * warps / t / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
