/*
 * cp_peaks.h -- libcppeaks.so: fp64 roofline denominators measured on the current device in the
 * benchmark's own run (bench.py).  A measurement helper beside libcp.so, not part of the hot
 * path: MEASURED_PEAKS.json provides the HBM copy bandwidth and bf16 tensor rate only, while the
 * restriction mode products (DMMA) and the R = 16 MTTKRP (near the fp64 ridge) need
 * the fp64 figures.
 *
 * cpp_fp64_peaks: best of `reps` CUDA-event-timed launches of
 *   - a DFMA kernel (8 independent fma chains per thread, 8 x 256-thread CTAs per SM)  -> TFLOP/s
 *   - a DMMA kernel (mma.sync.aligned.m8n8k4.f64, 8 independent accumulators per warp) -> TFLOP/s
 *   dfma_tflops, dmma_tflops  [host] outputs;  reps >= 1.
 *   Returns 0, -1 (bad argument) or -4 (CUDA error).  Synchronizes the device; uses the legacy
 *   default stream; allocates 8 bytes of device memory for the duration of the call.
 *
 * cpp_launch_floor_us: n back-to-back launches of an empty 1-CTA kernel on the legacy default
 *   stream, device time per launch in microseconds (CUDA events) -> *us_per_launch [host].
 *   The launch floor of the latency-bound small configurations (c0-c2).
 *   Returns 0, -1 (n < 1 or null output) or -4.
 */
#ifndef CP_PEAKS_H
#define CP_PEAKS_H
#ifdef __cplusplus
extern "C" {
#endif
int cpp_fp64_peaks(double *dfma_tflops, double *dmma_tflops, int reps);
int cpp_launch_floor_us(int n, double *us_per_launch);
#ifdef __cplusplus
}
#endif
#endif
