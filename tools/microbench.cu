// Microbenchmarks for the B200 fp64 roofline denominators that MEASURED_PEAKS.json lacks:
//  - DFMA throughput (fp64 vector pipe)
//  - DMMA throughput (mma.sync m8n8k4 f64, legacy fp64 tensor path)
//  - read-only HBM stream bandwidth (MTTKRP reads Z once; no write stream)
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} }while(0)

template<int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0; for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 123.456) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0001;
  double d[8][2];
  for (int c = 0; c < 8; ++c) { d[c][0] = c; d[c][1] = c + 1; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
  if (s == 123.456) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ x, size_t n2, double* out) {
  double s0 = 0, s1 = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
    double2 v = __ldg(&x[i]); s0 += v.x; s1 += v.y;
  }
  if (s0 + s1 == 123.456) out[0] = s0;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s SMs %d L2 %d MB\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  // DFMA
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 20000, threads = 256, blocks = sms * 8;
    dfma_kernel<8><<<blocks, threads>>>(out, 10, 1.0000001, 1e-9);
    CK(cudaEventRecord(e0));
    dfma_kernel<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)threads * blocks;
    printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 20000, threads = 256, blocks = sms * 8;
    CK(cudaEventRecord(e0));
    dmma_kernel<<<blocks, threads>>>(out, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (threads / 32) * (double)blocks;
    printf("DMMA m8n8k4: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  size_t bytes = (size_t)2 << 30; double2* x; CK(cudaMalloc(&x, bytes)); CK(cudaMemset(x, 0, bytes));
  for (int cfg = 0; cfg < 4; ++cfg) {
    int blocks = sms * (cfg + 1) * 2, threads = 512;
    read_kernel<<<blocks, threads>>>(x, bytes / 16, out);
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(e0)); read_kernel<<<blocks, threads>>>(x, bytes / 16, out);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("read-only stream (%d blocks x %d): %.1f GB/s\n", blocks, threads, bytes / best / 1e6);
  }
  CK(cudaGetLastError());
  return 0;
}
