// probe_tma_ring.cu -- what a minimal cp.async.bulk ring can stream from HBM: 296 CTAs (2 per SM),
// one producer warp issuing `ncopy` bulk copies of `cbytes` per stage into an `nst`-stage ring, one
// consumer warp that only hands the stages back.  Each CTA streams its own contiguous range of a
// 1 GiB buffer (the streaming kernels' pattern).  Prints GB/s per (copy size, stage size, depth).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t *b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(n)); }
__device__ __forceinline__ void mb_expect(uint64_t *b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t *b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory"); }
__device__ __forceinline__ bool mb_try(uint64_t *b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(s32(b)), "r"(ph) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mb_wait(uint64_t *b, uint32_t ph) { while (!mb_try(b, ph)) {} }
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s32(dst)), "l"(src), "r"(bytes), "r"(s32(bar)) : "memory");
}

__global__ void __launch_bounds__(64, 2) ring(const char *z, long total, int cbytes, int ncopy, int nst, int dstpad) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t full[8], empty[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long sbytes = (long)cbytes * ncopy;
  const long per = total / gridDim.x / 65536 * 65536;  // aligned per-CTA range
  const long r0 = per * blockIdx.x, nstage = per / sbytes;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int st = 0; uint32_t ph = 0;
  if (warp == 0) {
    for (long i = 0; i < nstage; ++i) {
      mb_wait(&empty[st], ph ^ 1u);
      if (lane == 0) mb_expect(&full[st], (uint32_t)sbytes);
      __syncwarp();
      char *dst = sm + (long)st * (sbytes + (long)ncopy * dstpad);
      for (int c = lane; c < ncopy; c += 32) bulk(dst + (long)c * (cbytes + dstpad), z + r0 + i * sbytes + (long)c * cbytes, cbytes, &full[st]);
      if (++st == nst) { st = 0; ph ^= 1u; }
    }
  } else {
    for (long i = 0; i < nstage; ++i) {
      mb_wait(&full[st], ph);
      if (lane == 0) mb_arrive(&empty[st]);
      __syncwarp();
      if (++st == nst) { st = 0; ph ^= 1u; }
    }
  }
}

int main() {
  const long total = 1L << 30;
  char *z; cudaMalloc(&z, total); cudaMemset(z, 0, total);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](int cbytes, int ncopy, int nst, int pad) {
    const size_t smem = (size_t)nst * ncopy * (cbytes + pad);
    if (smem > 108 * 1024) return;
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(e0); ring<<<296, 64, smem>>>(z, total, cbytes, ncopy, nst, pad); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    const long per = total / 296 / 65536 * 65536;
    const long moved = per / ((long)cbytes * ncopy) * ((long)cbytes * ncopy) * 296;
    printf("copy %6d B x %3d = stage %6ld B, %d stages (%3zu KB/CTA), dst pad %3d: %7.1f us  %5.0f GB/s  %s\n", cbytes, ncopy,
           (long)cbytes * ncopy, nst, smem >> 10, pad, best * 1e3, moved / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  run(2048, 24, 2, 32);   // the c4a plan: 24 columns of 2 KB, 2 stages, padded destination
  run(2048, 24, 2, 0);
  run(2048, 12, 4, 32);
  run(2048, 8, 6, 32);
  run(2048, 4, 8, 32);
  run(4096, 12, 2, 0);
  run(8192, 6, 2, 0);
  run(49152, 1, 2, 0);
  run(24576, 1, 4, 0);
  run(16384, 1, 6, 0);
  run(8192, 1, 8, 0);
  run(32768, 1, 3, 0);
  run(1024, 48, 2, 0);
  run(768, 32, 4, 32);    // c4b-like columns (96 rows)
  return 0;
}
