// cp_internal.cuh -- shared device helpers and launch plans of libcp.so (sm_100a).
// Product code: nothing here is shared with, or derived from, oracle/.
#pragma once
#include <cstdint>
#ifdef CP_CTA_TIMELINE
#include <cstdio>
#endif
#include <utility>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/cp.h"

namespace cpk {

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;   // 256 consumer threads
constexpr int kStreamThreads = kConsumers + 64;   // + TMA producer warp + weight warp
constexpr int kMaxRows = 512;                     // widest row block (V = 2: 2 rows / thread)
constexpr int kMaxDigits = CP_MAX_N - 1;          // column multi-index digits (modes 1..N-1)

// OP_YL: the first pass of the dimension-tree sweep -- the mode-1 contraction of Z with the
// Khatri-Rao rows of modes 2..N-1, written per i_1 segment as an I_0 x R block (no contraction
// with A^(0)); see stream_kernel.cuh.
enum StreamOp { OP_MTTKRP = 0, OP_RESID = 1, OP_YL = 2 };

// Gamma^(mode) factorization job (gamma_job.cuh): Upsilon^(k) for k != mode is the sum of cnt[k]
// R x R partials at src[k] (stride R*R, summed in order, total written to ups[k]) or, cnt[k] = 0,
// the total at src[k]; out: L^{-1} (R x R row-major) in linv; CP_ENOTSPD + mode in status.
// gram_rows > 0 (stream_mma.cuh gram_rows_warp, before the job): Upsilon^(gram_mode) is first
// formed from the gram_rows rows of the row-major factor copy gram_At (row stride gram_RS) and
// written to ups -- the Gram the previous sweep's in-pass tail solve deferred (TailSolve::fin = 0).
struct GammaJob {
  int on, N, R, mode;
  const double *src[CP_MAX_N];
  int cnt[CP_MAX_N];
  double *ups, *linv, *status;
  int gram_mode, gram_RS;
  int64_t gram_rows;
  const double *gram_At;
};

// The sweep's last solve inside the last streaming pass (N = 3 dimension-tree sweep, MMA plans;
// stream_mma.cuh sweep_tail): the last contributor of each segment i_2 (tagged ticket) sums the
// segment's partials into row i_2 of M^(2), solves x = L^{-T}(L^{-1}(m + f)) in one warp
// (lane = component; eq:relaxinnersolve, reading R1) and writes the row of A^(2), At^(2) and the
// row's <M,A>, <F,A>; the last CTA of the grid (ticket gtick) forms Upsilon^(2) over all rows in
// a fixed order and f, f~ (readings R5, R6).  L^{-1} comes from this launch's Gamma job (CTA 0's
// weight warp), published through the flag gjflag.  No solve launch follows.
struct TailSolve {
  int on;
  int fin;                 // 1: the last CTA forms Upsilon^(2) and f, f~ (the call's last sweep);
                           // 0: rows only -- the next sweep's Gamma^(0) job forms Upsilon^(2)
                           // (GammaJob::gram_rows) and this sweep's f is not evaluated
  int dot_stride;          // stride between the modes' <F,A> partial arrays
  int nsolve[2];           // <F,A> partials of modes 0, 1 (their solves' grid sizes)
  const double *linv;      // L^{-1} of Gamma^(2), R x R row-major (Gamma job of this launch)
  const double *F;         // F^(2) or null
  double *A, *At;          // A^(2) column-major; row-major copy (stride RS)
  double *rowdot;          // workspace: per row <M,A> [0, In) and <F,A> [In, 2 In)
  const double *dotF;      // <F,A> partials of the earlier modes
  double *Ups;             // N x R x R Gram totals
  const double *normZ2;
  double *status, *out;
  // u32 completion words, zeroed by the prep kernel and reset by their last users: one ticket
  // per segment i_2, the grid ticket, the Gamma job's "done" flag
  unsigned *segtick, *gtick, *gjflag;
};

// doubles of shared memory sweep_tail needs: L^{-1}, the block sums, and (after them) one
// (8 NT)^2 Gram tile per consumer warp
__host__ __device__ constexpr int sweep_tail_fixed_doubles(int R) { return R * (R + 1) + 24; }
__host__ __device__ constexpr int sweep_tail_doubles(int R) {
  return sweep_tail_fixed_doubles(R) + kConsumerWarps * (8 * ((R + 7) / 8)) * (8 * ((R + 7) / 8));
}

// Plan of one streaming pass over Z (MTTKRP of one mode, or the residual pass of cp_fit).
// Z is viewed as an I1 x Q column-major matrix (Q = P / I1 "columns" = mode-1 fibers).
// Column groups: CTA (c, rb) streams virtual columns [v0(c), v1(c)) restricted to row block
// rb.  For mode m >= 1 the virtual order puts i_m outermost, so that a contiguous v-range
// touches few output rows ("segments" of Qn columns each).
struct StreamPlan {
  int N, R, mode, op;
  int V;            // rows per consumer thread: 8/4/2 (I1 divisible), 1 (odd I1: scalar fallback)
  int Wmax;         // row-block width (even when V = 2)
  int RB;           // number of row blocks
  int Gc;           // number of column groups
  int cps;          // columns per pipeline stage
  int nstages;      // pipeline depth
  int slots;        // mode >= 1: output segments a column group can touch
  int smem_bytes;
  int RS;           // row stride of the row-major factor copies At (R rounded up to even)
  int64_t dims[CP_MAX_N];
  int64_t I1, Q;    // rows and columns of the mode-1 view
  int64_t Qn;       // columns per segment (mode >= 1); Q for mode 0 / residual
  int64_t L;        // contiguous run length in q for one segment (prod_{0<k<m} I_k); Q for mode 0
  int64_t In;       // I_mode (segments); 1 for mode 0 / residual
  // v-order odometer: digit j (fastest first) is the index of mode ord[j], radix rad[j],
  // column stride qsd[j] = prod_{1 <= k < ord[j]} I_k.  mode 0: modes 1..N-1;
  // mode m >= 1: modes 1..m-1, m+1..N-1, then m (the segment digit).
  int nd;
  int ord[CP_MAX_N - 1];
  int rad[CP_MAX_N - 1];
  int64_t qsd[CP_MAX_N - 1];
  const double *Z;
  const double *At[CP_MAX_N];   // row-major (I_k x R) copies of the factors
  double *part;     // partial outputs (workspace)
  double *yl;       // OP_YL: I0 x R block per fully owned segment (segment-major)
  double *edge;     // OP_YL: per CTA 2 blocks for partially owned segments
  unsigned *segcnt; // OP_YL (MMA): per (segment, row block) completion tickets (zeroed by prep), or null
  int red_doubles;  // consumers' shared reduction area (doubles)
  // FP64 tensor-core consumers (stream_mma.cuh): mma = 1 selects stream_mma_kernel<NT, MT, OP>
  int mma;
  int ks, mt, nt;   // k-split groups, m-tiles (8 rows) per warp, n-tiles (8 ranks)
  int zcs;          // shared-memory column stride of a Z stage (doubles); 0: the block width Wb
  int zst;          // doubles per Z stage in shared memory
  int direct_w;     // Khatri-Rao rows are the staged factor rows (no weight warp)
  int ars, wstr;    // shared-memory row strides of the staged factor rows / the weight rows
  int srows;        // the producer also stages the slow digits' factor rows (kMaxDigits per stage)
  GammaJob gj;      // optional side job for the idle weight warp of CTA 0 (MMA kernel, direct_w)
  int gjsm;         // shared-memory doubles reserved for it
  int64_t keep_q;   // L2 residency across passes: Z columns q < keep_q are fetched with an
                    // evict_last policy, the rest evict_first (0: no hints).  See DESIGN 6.8.
  int prefetch;     // the launch's predecessor does not write Z: the producer issues the Z part of
                    // its first nstages stages before the PDL wait (stream_kernel.cuh produce)
  int dbg;          // experiments only (knob CP_STREAM_DBG, -DCP_EXPERIMENTS builds): 1 = consumers skip the FMAs
  // MMA plans whose row block is the whole column (RB = 1): one 3-D tensor-map TMA per full
  // stage instead of one bulk copy per column.  View {I1, qsd[0], Q / qsd[0]} of Z, box
  // {zcs, 1, cps}: the stage's columns are consecutive along dim 2, and the box rows past I1
  // are out of bounds -> zero-filled padding of the zcs column slots (no extra HBM bytes).
  int use_tmap;
  int astage;       // doubles per stage of the staged factor rows (abuf)
  int srs;          // doubles per staged slow-digit row slot (sbuf)
  int sstr;         // rank stride inside a slow-row slot (1; fcm: 2 -- a {2, R} box, TMA needs
                    // 16-byte box rows)
  // cp_mttkrp (MMA plans, direct_w): fcm = 1 -- the producer stages the factor rows straight
  // from the caller's column-major factors Af through 2-D tensor maps (fmap[0]: box {fs, R} of
  // A^(ord[0]), landing rank-major [R][fs], fs = 4 mod 16 doubles for conflict-free B
  // fragments; fmap[j], j >= 1: box {2, R} of the slow digit j's factor), so no prep launch
  // (row-major At copies) precedes the pass; the mode >= 1 epilogue reads A^(1) from Af[0].
  int fcm, fs;
  const double *Af[CP_MAX_N];
  // cp_mttkrp in one launch (MMA plans, OP_MTTKRP): Mout != null -- the pass finishes M itself.
  // Modes >= 1: the last contributor of each segment (tagged ticket tick[segment]) sums the
  // segment's partials in the fixed order of reduce_mttkrp_kernel; mode 0: a grid barrier
  // (tick[0..2]), then every CTA sums a slice of the I1 x R entries in the order of
  // reduce_mode0_kernel.  tag: this launch's nonce (tagged_arrive).
  double *Mout;
  unsigned long long *tick;
  unsigned tag;
  TailSolve tail;   // the sweep's last solve + finalize inside this pass (see TailSolve)
  alignas(64) CUtensorMap tmap;
  alignas(64) CUtensorMap fmap[kMaxDigits];
};

// Kernel table: one entry per (R, V, op) instantiation of stream_kernel.
struct StreamEntry {
  cudaError_t (*launch)(const StreamPlan &, cudaStream_t);
  const void *kernel;
};
constexpr int stream_index(int R, int V, int op) {
  return (R * 4 + (V == 8 ? 3 : (V == 4 ? 2 : V - 1))) * 3 + op;
}
// Consumer rank tile (see StreamTile in stream_kernel.cuh): ranks per thread and rank groups.
__host__ __device__ constexpr int stream_rg(int R, int op) { return (op != 1 && R > 12) ? (R + 7) / 8 : 1; }
__host__ __device__ constexpr int stream_rt(int R, int op) {
  return (stream_rg(R, op) > 1 && (((R + stream_rg(R, op) - 1) / stream_rg(R, op)) & 1))
             ? (R + stream_rg(R, op) - 1) / stream_rg(R, op) + 1
             : (R + stream_rg(R, op) - 1) / stream_rg(R, op);
}
// shared-memory reduction area of the consumers (doubles)
__host__ __device__ constexpr int stream_red_doubles(int R, int op) { return 256 * stream_rt(R, op) + 8 > 8 * R + 8 ? 256 * stream_rt(R, op) + 8 : 8 * R + 8; }
constexpr int kStreamTableSize = stream_index(CP_MAX_R, 8, 2) + 1;
void register_stream_part0(StreamEntry *t);
void register_stream_part1(StreamEntry *t);
void register_stream_part2(StreamEntry *t);
void register_stream_part3(StreamEntry *t);
const StreamEntry &stream_entry(int R, int V, int op);
// FP64 tensor-core variants stream_mma_kernel<NT, MT, OP> (OP_MTTKRP, OP_YL, OP_RESID)
constexpr int mma_index(int nt, int mt, int op) {
  return ((nt - 1) * 8 + (mt - 1)) * 3 + (op == OP_YL ? 1 : (op == OP_RESID ? 2 : 0));
}
constexpr int kMmaTableSize = mma_index(4, 8, OP_RESID) + 1;
void register_stream_mma(StreamEntry *t);    // lean kernels (FEAT = false)
void register_stream_mma_f(StreamEntry *t);  // full-feature kernels
const StreamEntry &stream_mma_entry(int nt, int mt, int op, bool feat = true);

// ---------------------------------------------------------------- host configuration
// Path selectors (documented in include/cp.h): environment switches between result-equivalent
// code paths that the parity tests cover (e.g. CP_STREAM_MMA=0: DFMA consumers).  Read on every
// call (nothing cached).  Any other variable name is rejected (returns dflt).
int path_flag(const char *name, int dflt);
// Tuning and debugging knobs (stage sizes, ring depth, kernel-skip masks ...): read from the
// environment ONLY in a library built with -DCP_EXPERIMENTS (tools/); the shipped library
// always uses the defaults, so no environment variable can change what it computes.
int knob(const char *name, int dflt);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel, bytes).
cudaError_t ensure_smem_attr(const void *kernel, int bytes);
int current_device();

// Host: build the plan (geometry only; pointers filled by the caller).
bool make_stream_plan(StreamPlan &p, const cp_shape &s, int mode, int op, int num_sms, bool fcm = false);
size_t stream_part_doubles(const StreamPlan &p);
cudaError_t launch_stream(const StreamPlan &p, cudaStream_t st);

// Programmatic dependent launch (PDL): the sweep's kernels are launched with programmatic
// stream serialization, so a kernel's blocks are scheduled while its predecessor runs.  Every
// kernel launched that way starts with griddep(): wait until the predecessor grid has completed
// and its writes are visible (before any global access to data a predecessor may write and before
// any early return, so completion stays transitive along the stream), THEN allow the next kernel
// to launch.  Because the trigger follows the wait, a kernel's blocks only start once everything
// up to its predecessor's predecessor is complete: code before griddep() may read data that the
// immediate predecessor does not write (the Z prefetch of the streaming kernels,
// StreamPlan::prefetch).
__device__ __forceinline__ void griddep() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Timing builds only (-DCP_CTA_TIMELINE, tools/sweep_timeline.py): every block's thread 0 prints
// its entry time, the time its griddep() wait returned and its exit time (globaltimer, ns).
#ifdef CP_CTA_TIMELINE
__device__ __forceinline__ unsigned long long ctl_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CTL_BEGIN const unsigned long long ctl_e = ctl_clock();
#define CTL_AFTER_WAIT const unsigned long long ctl_w = ctl_clock();
#define CTL_END(tag)                                                                                   \
  if (threadIdx.x == 0)                                                                                \
    printf("CTK %s %d %llu %llu %llu\n", tag, (int)blockIdx.x, ctl_e, ctl_w, ctl_clock());
#else
#define CTL_BEGIN
#define CTL_AFTER_WAIT
#define CTL_END(tag)
#endif

// PDL per launch class (env CP_PDL_MASK, bit c = class c; CP_PDL=0 clears all):
//   kPdlStream: the Z-streaming kernels, kPdlCluster: ylsolve (8-CTA clusters), kPdlSmall: the rest,
//   kPdlWide: 1024-thread reduction kernels (off by default: launched early, their waiting CTAs
//   took the SM slots the streaming pass before them could use)
enum { kPdlStream = 0, kPdlCluster = 1, kPdlSmall = 2, kPdlWide = 3 };
bool pdl_enabled(int cls = kPdlSmall);
template <typename... KArgs, typename... Args>
cudaError_t launch_kc(int cls, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled(cls) ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a pipeline bug must fail loudly (trap -> cudaErrorLaunchFailure) instead of
// hanging the GPU.  ~30 s at 2 GHz is far beyond any legitimate wait.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(bar, parity)) {
    if (clock64() - t0 > 60000000000LL) __trap();
  }
}
// TMA bulk copy global -> shared (async proxy), completion via mbarrier transaction bytes.
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 2-D tensor-map TMA (box -> shared memory, complete_tx on the stage barrier)
__device__ __forceinline__ void tma_load_2d(void *dst_smem, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst_smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// 3-D tensor-map TMA (box -> shared memory, complete_tx on the stage barrier)
__device__ __forceinline__ void tma_load_3d(void *dst_smem, const CUtensorMap *map, int c0, int c1, int c2,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst_smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_hint(void *dst_smem, const CUtensorMap *map, int c0, int c1, int c2,
                                                 uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(
          smem_u32(dst_smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// The same copy with an L2 eviction-priority policy (createpolicy; evict_last / evict_first).
__device__ __forceinline__ void bulk_g2s_hint(void *dst_smem, const void *src_gmem, uint32_t bytes,
                                              uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// Opaque copy of a value: address arithmetic derived from it inside a rarely taken branch
// (the per-segment flushes of stream_kernel) cannot be hoisted out of the streaming loop,
// where it would pin registers and force spills.
__device__ __forceinline__ int opaque(int x) {
  int y;
  asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ int64_t opaque(int64_t x) {
  int64_t y;
  asm volatile("mov.b64 %0, %1;" : "=l"(y) : "l"(x));
  return y;
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- in-kernel completion
// Tagged arrival counters over caller-owned, uninitialized workspace: a 64-bit word holds
// (tag << 32 | count).  An arrival whose tag differs from the word's starts a new count (no
// zeroing launch needed); the last of n arrivals of a launch resets the word to 0.  Tags are
// per-launch host nonces, never 0, so a word left by a completed launch never matches, and a CUDA
// graph that replays one tag starts every replay from 0.  Called by one thread; returns true for
// the last arrival.  The caller fences its data stores before arriving.
__device__ __forceinline__ bool tagged_arrive(unsigned long long *w, unsigned tag, unsigned n) {
  const unsigned long long hi = (unsigned long long)tag << 32;
  unsigned long long cur = *reinterpret_cast<volatile unsigned long long *>(w);
  for (;;) {
    const unsigned long long nv = ((cur & 0xffffffff00000000ull) == hi) ? cur + 1 : (hi | 1ull);
    const unsigned long long prev = atomicCAS(w, cur, nv);
    if (prev == cur) {
      if ((unsigned)nv != n) return false;
      atomicExch(w, 0ull);
      return true;
    }
    cur = prev;
  }
}
// Grid-wide barrier of a co-resident grid over words b[0..2] of uninitialized workspace.
// Arrivals count with atomicAdd (a CAS per arrival serializes a whole grid behind one address):
// CTA 0 first claims b[0] (arrivals) and b[2] (departures) for its tag -- grid_claim, after its
// griddep() wait, so the previous launch is done with them; an arrival that lands before the
// claim (seen as a foreign tag; the claim overwrites it) waits for the claim and arrives again.
// The last arrival resets b[0] and publishes the tag in b[1]; the others poll b[1].
// grid_depart (once the CTA no longer needs the barrier): the last CTA out clears b[1], so the
// next launch -- or graph replay of this one -- waits again.  Bounded: a grid that is not
// co-resident traps (cudaErrorLaunchFailure) instead of hanging the GPU.
__device__ __forceinline__ void grid_claim(unsigned long long *b, unsigned tag) {
  const unsigned long long mine = (unsigned long long)tag << 32;
  for (int i = 0; i < 3; i += 2) {
    unsigned long long cur = *reinterpret_cast<volatile unsigned long long *>(b + i);
    while ((cur & 0xffffffff00000000ull) != mine) {
      const unsigned long long prev = atomicCAS(b + i, cur, mine);
      if (prev == cur) break;
      cur = prev;
    }
  }
}
__device__ __forceinline__ bool counted_arrive(unsigned long long *w, unsigned tag, unsigned n) {
  const long long t0 = clock64();
  for (;;) {
    const unsigned long long old = atomicAdd(w, 1ull);
    if ((unsigned)(old >> 32) == tag) {
      if ((unsigned)old + 1u != n) return false;
      atomicExch(w, 0ull);
      return true;
    }
    while ((unsigned)(*reinterpret_cast<volatile unsigned long long *>(w) >> 32) != tag) {
      __nanosleep(64);
      if (clock64() - t0 > 20000000000LL) __trap();
    }
  }
}
__device__ __forceinline__ void grid_barrier(unsigned long long *b, unsigned tag, unsigned n) {
  if (counted_arrive(b, tag, n)) {
    __threadfence();
    atomicExch(b + 1, (unsigned long long)tag);
    return;
  }
  const volatile unsigned long long *rel = b + 1;
  const long long t0 = clock64();
  while (*rel != (unsigned long long)tag) {
    __nanosleep(64);
    if (clock64() - t0 > 20000000000LL) __trap();
  }
  __threadfence();
}
__device__ __forceinline__ void grid_depart(unsigned long long *b, unsigned tag, unsigned n) {
  if (counted_arrive(b + 2, tag, n)) atomicExch(b + 1, 0ull);
}

}  // namespace cpk
