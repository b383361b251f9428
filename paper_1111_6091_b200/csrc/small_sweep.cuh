// Fused multi-sweep ALS / BNGS kernel for tensors resident in one CTA's shared memory
// (small_sweep.cu).  Used by cp_als_sweep / cp_als_sweeps when small_sweep_smem_bytes() != 0.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "../../include/cp.h"

namespace cpk {

constexpr int kSmallSweepThreads = 512;
constexpr int kSmallSweepMaxR = 32;
constexpr int64_t kSmallSweepMaxP = 16384;  // 128 KiB of Z: one CTA streams it faster than ~8 launches

struct SmallSweepArgs {
  int N, R, nsweeps;
  int64_t P, imax, npart, lr;  // lr: max over modes of left + right (Khatri-Rao halves)
  int64_t dims[CP_MAX_N];
  const double *Z, *normZ2;
  double *A[CP_MAX_N];
  const double *F[CP_MAX_N];
  double *out;
  int grad;               // 1: cp_gradient at this iterate (no updates): gout = f, g, ||G^(n)||^2
  int normalize;          // 1: eq:ALSnorm (no sort) after every sweep (CP_SWEEPS_NORMALIZE)
  int grad_after;         // 1: after the nsweeps sweeps, the gradient pass at the new iterate in the
                          // same launch (cp_als_sweeps_then_gradient): out as the sweeps, gout as cp_gradient
  double *G[CP_MAX_N];    // gradient pass: G^(n) outputs (entries may be null)
  const double *gF[CP_MAX_N];  // gradient pass: F entering G (R21), or null
  double *gout;           // gradient pass: 2 + N doubles
};

// Single-warp variant for the tiniest tensors (tiny_sweep.cu): sweeps only (no gradient mode)
constexpr int kTinySweepMaxR = 4;
constexpr int64_t kTinySweepMaxP = 512;
bool tiny_sweep_ok(const cp_shape &s);
cudaError_t launch_tiny_sweep(const cp_shape &s, const double *Z, const double *normZ2, double *const *A,
                              const double *const *F, int nsweeps, double *out, cudaStream_t st, bool normalize);

// dynamic shared memory the kernel needs for shape s, or 0 if s is not small enough
size_t small_sweep_smem_bytes(const cp_shape &s);
cudaError_t launch_small_sweep(const cp_shape &s, const double *Z, const double *normZ2, double *const *A,
                               const double *const *F, int nsweeps, double *out, cudaStream_t st,
                               double *const *G = nullptr, bool grad = false, bool normalize = false,
                               double *gout = nullptr, const double *const *gF = nullptr);

}  // namespace cpk
