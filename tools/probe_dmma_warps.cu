// probe_dmma_warps.cu -- DMMA (mma.sync m8n8k4 f64) throughput against resident warps per SM
// sub-partition and independent accumulators per warp: how much latency hiding the FP64 tensor
// path needs (sizing of the mode-product GEMM's warp tiles / CTAs per SM).
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void k(double *out, int iters) {
  const double a = threadIdx.x * 1e-3, b = 1.0001;
  double d[ACC][2];
#pragma unroll
  for (int c = 0; c < ACC; ++c) { d[c][0] = c; d[c][1] = c + 1; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < ACC; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < ACC; ++c) s += d[c][0] + d[c][1];
  if (s == 123.456) out[0] = s;
}

template <int ACC>
static void run(double *out, int sms, int warps_per_sm) {
  const int iters = 4000 * 16 / ACC;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(e0); k<ACC><<<sms, 32 * warps_per_sm>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  const double fl = 2.0 * 8 * 8 * 4 * ACC * (double)iters * warps_per_sm * sms;
  printf("acc/warp %2d  warps/SM %2d (%.1f per sub-partition): %.1f TFLOP/s\n", ACC, warps_per_sm, warps_per_sm / 4.0, fl / best / 1e9);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out; cudaMalloc(&out, 8);
  k<8><<<sms, 256>>>(out, 10); cudaDeviceSynchronize();
  for (int w : {4, 8, 16, 32}) { run<1>(out, sms, w); run<2>(out, sms, w); run<4>(out, sms, w); run<8>(out, sms, w); run<16>(out, sms, w); run<32>(out, sms, w); }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
