// capi.cu -- the C ABI of libcp.so (include/cp.h): argument validation, workspace layout,
// launch plans and the launch sequences of cp_mttkrp / cp_als_sweep / cp_fit / cp_norm2 /
// cp_mode_product.  Every numeric step runs in the CUDA kernels of this directory.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <chrono>
#include <memory>
#include <mutex>
#include <vector>

#include <cudaTypedefs.h>

#include "gamma_job.cuh"
#include "mg_kernels.cuh"
#include "small_sweep.cuh"
#include "small_kernels.cuh"
#include "stream_kernel.cuh"

namespace cpk {
cudaError_t launch_mode_product(int N, const int64_t *dims, const double *Z, int mode,
                                const double *U, int64_t J, double *X, cudaStream_t st);
int mode_product_launch_count(int N, const int64_t *dims, int mode);

static thread_local int g_launches = 0;

// ---------------------------------------------------------------- kernel table
static StreamEntry g_table[kStreamTableSize];
static std::once_flag g_table_once;

const StreamEntry &stream_entry(int R, int V, int op) {
  std::call_once(g_table_once, [] {
    register_stream_part0(g_table);
    register_stream_part1(g_table);
    register_stream_part2(g_table);
    register_stream_part3(g_table);
  });
  return g_table[stream_index(R, V, op)];
}

static StreamEntry g_mma_table[2][kMmaTableSize];  // [0]: lean kernels, [1]: full-feature kernels
static std::once_flag g_mma_once;

const StreamEntry &stream_mma_entry(int nt, int mt, int op, bool feat) {
  std::call_once(g_mma_once, [] {
    register_stream_mma(g_mma_table[0]);
    register_stream_mma_f(g_mma_table[1]);
  });
  return g_mma_table[feat ? 1 : 0][mma_index(nt, mt, op)];
}

// Does the plan use anything the lean instantiation leaves out (stream_kernel.cuh, P_FCM)?
static bool stream_mma_feat(const StreamPlan &p) {
  return p.fcm != 0 || p.prefetch != 0 || p.tail.on != 0 || p.Mout != nullptr || (p.gj.on && p.gj.gram_rows > 0);
}

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  return dev;
}

static int device_sms() {
  static std::mutex mu;
  static int cached[64] = {0};
  const int dev = current_device();
  {
    std::lock_guard<std::mutex> lk(mu);
    if (dev >= 0 && dev < 64 && cached[dev] > 0) return cached[dev];
  }
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) return 148;
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= 0 && dev < 64) cached[dev] = sms;
  return sms;
}

static int parse_env(const char *name, int dflt) {
  const char *v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

int path_flag(const char *name, int dflt) {
  static const char *const kPaths[] = {"CP_STREAM_MMA", "CP_RESID_MMA", "CP_STREAM_TMAP", "CP_SMALL_SWEEP", "CP_MTTKRP_FCM", "CP_MTTKRP_FUSED", "CP_MODEPROD_PIPE", "CP_SWEEP_TAIL", "CP_TINY_SWEEP", "CP_STREAM_PREFETCH", "CP_STREAM_LEAN", "CP_SWEEPS_GRAD_FUSED",
                                       "CP_SWEEP_TREE", "CP_YLSOLVE", "CP_MODEPROD_DMMA", "CP_MG_GRAPH",
                                       "CP_ALS_GRAPH", "CP_MG_STRUCTURED", "CP_PDL"};
  for (const char *k : kPaths)
    if (strcmp(k, name) == 0) return parse_env(name, dflt);
  return dflt;
}

int knob(const char *name, int dflt) {
#ifdef CP_EXPERIMENTS
  return parse_env(name, dflt);
#else
  (void)name;
  return dflt;
#endif
}

cudaError_t ensure_smem_attr(const void *kernel, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, const void *>, int>> done;
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(mu);
  for (const auto &d : done)
    if (d.first.first == dev && d.first.second == kernel && d.second >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  for (auto &d : done)
    if (d.first.first == dev && d.first.second == kernel) {
      d.second = bytes;
      return cudaSuccess;
    }
  done.push_back({{dev, kernel}, bytes});
  return cudaSuccess;
}

// measured (tools/time_sweep.py, no profiling events): PDL on the 8-CTA-cluster ylsolve launches cost
// c4a ~15 us per sweep (its CTAs, launched early, wait where the pass could run); default: stream +
// small kernels.  CP_PDL=0 (path selector) disables PDL everywhere; the mask is an experiment knob.
constexpr int kPdlDefaultMask = (1 << kPdlStream) | (1 << kPdlSmall);
// Launch nonces of the tagged completion words (cp_internal.cuh tagged_arrive): never 0, seeded
// per process so a workspace handed between processes does not meet its previous tags.
static unsigned next_tag() {
  static std::atomic<unsigned> ctr{(unsigned)std::chrono::steady_clock::now().time_since_epoch().count() * 2654435761u};
  unsigned t;
  do t = ctr.fetch_add(1u); while (t == 0u || t == 0xffffffffu);
  return t;
}

bool pdl_enabled(int cls) {
  const int mask = path_flag("CP_PDL", 1) != 0 ? knob("CP_PDL_MASK", kPdlDefaultMask) : 0;
  return (mask >> cls) & 1;
}

// resident CTAs / SM of a streaming kernel at a dynamic smem size; cached per (device, kernel,
// smem) (the CUDA queries cost microseconds, and every call plans its launches)
static int kernel_occupancy(const void *kernel, int smem) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void *, int>, std::pair<int, int>>> cache;
  const int dev = current_device();
  {
    std::lock_guard<std::mutex> lk(mu);
    for (const auto &c : cache)
      if (c.first.first == kernel && c.first.second == smem && c.second.first == dev) return c.second.second;
  }
  int n = 0;
  if (ensure_smem_attr(kernel, 200 * 1024) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, kStreamThreads, smem) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  n = n > 0 ? n : 1;
  std::lock_guard<std::mutex> lk(mu);
  cache.push_back({{kernel, smem}, {dev, n}});
  return n;
}
static int stream_occupancy(int R, int V, int op, int smem) {
  return kernel_occupancy(stream_entry(R, V, op).kernel, smem);
}
static int stream_mma_occupancy(int nt, int mt, int op, int smem) {
  return kernel_occupancy(stream_mma_entry(nt, mt, op).kernel, smem);
}

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// v-order digits (see StreamPlan); false if a radix does not fit 32 bits
static bool plan_digits(StreamPlan &p, const cp_shape &s) {
  int64_t qstride[CP_MAX_N];
  qstride[1] = 1;
  for (int k = 2; k < s.N; ++k) qstride[k] = qstride[k - 1] * s.dims[k - 1];
  int j = 0;
  for (int k = 1; k < s.N; ++k)
    if (k != p.mode) p.ord[j++] = k;
  if (p.mode != 0) p.ord[j++] = p.mode;
  p.nd = j;
  for (int t = 0; t < p.nd; ++t) {
    if (s.dims[p.ord[t]] > 0x7fffffff) return false;
    p.rad[t] = (int)s.dims[p.ord[t]];
    p.qsd[t] = qstride[p.ord[t]];
  }
  return true;
}

// FP64 tensor-core consumer geometry (stream_mma.cuh): row block, k-split and m-tiles per warp
static bool plan_mma_ok(const StreamPlan &p, const cp_shape &s, int op) {
  return !(path_flag("CP_STREAM_MMA", 1) == 0 || (op == OP_RESID && path_flag("CP_RESID_MMA", 1) == 0) || s.R > 32 ||
           (p.I1 & 1));
}
// row block = the whole (even) column, padded column slots within the TMA box limit: the stage
// can be one tensor-map TMA whose out-of-bounds rows fill the padding (launch_stream)
static bool tmap_geometry_ok(const StreamPlan &p) {
  return p.mma && p.RB == 1 && p.zcs > p.I1 && p.zcs <= 256 && (p.I1 & 1) == 0 && p.V >= 2;
}

static bool plan_mma(StreamPlan &p, const cp_shape &s, int op) {
  if (!plan_mma_ok(p, s, op)) return false;
  p.nt = (s.R + 7) / 8;
  int mt_max = (p.nt <= 2) ? 8 : 4;
  const int mt_env = knob("CP_MMA_MTMAX", 4);  // measured: MT = 8 (64 accumulators) serializes the A loads
  if (mt_max > mt_env) mt_max = mt_env;
  int64_t Wt = p.I1;
  if (ceil_div(p.I1, 8) > 8 * mt_max) Wt = 64 * mt_max;
  p.RB = (int)ceil_div(p.I1, Wt);
  int64_t W = ceil_div(p.I1, p.RB);
  W = ceil_div(W, 8) * 8;
  p.Wmax = (int)W;
  const int mtiles = (int)(W / 8);
  double best = -1.0;
  for (int ks = 1; ks <= 8; ks *= 2) {
    const int wpg = kConsumerWarps / ks;
    const int mt = (mtiles + wpg - 1) / wpg;
    if (mt > mt_max) continue;
    const double eff = (double)mtiles * ks / (8.0 * mt) - 0.02 * (ks > 1);
    if (eff > best + 1e-9) {
      best = eff;
      p.ks = ks;
      p.mt = mt;
    }
  }
  if (best < 0) return false;
  p.mma = 1;
  p.V = 2;
  // column stride = 8 (mod 16) doubles.  (64-bit shared loads are served per half-warp, so = 4
  // (mod 16) is what makes the A-fragment reads conflict-free -- 2 wavefronts instead of 4, as in
  // the GEMM of mode_product.cu -- but the shared-memory pipe does not limit these kernels: with
  // = 4 the sweeps gained 0-0.7 %, while cp_mttkrp mode 0 on c4a went from 0.208 to 0.298 ms
  // (profiles/r02g_zcs_mode0.txt), so the stride stays; CP_ZCS_PAD in experiment builds.)
  p.zcs = (int)(ceil_div(W, 16) * 16 + knob("CP_ZCS_PAD", 8));
  // residual pass: Z is read at the C-fragment positions (row gq, columns 2 tq, 2 tq + 1);
  // a column stride = 2 (mod 8) doubles makes each half-warp hit 16 distinct bank pairs
  if (op == OP_RESID) p.zcs = (int)(ceil_div(W, 8) * 8 + 2);
  return true;
}

bool make_stream_plan(StreamPlan &p, const cp_shape &s, int mode, int op, int num_sms, bool fcm) {
  memset(&p, 0, sizeof(p));
  p.N = s.N;
  p.R = s.R;
  p.op = op;
  p.mode = (op == OP_RESID) ? 0 : mode;
  int64_t P = 1;
  for (int k = 0; k < s.N; ++k) {
    p.dims[k] = s.dims[k];
    P *= s.dims[k];
  }
  p.I1 = s.dims[0];
  p.Q = P / p.I1;
  if (p.mode == 0) {
    p.In = 1;
    p.Qn = p.Q;
    p.L = p.Q;
  } else {
    p.In = s.dims[mode];
    p.Qn = p.Q / p.In;
    int64_t L = 1;
    for (int k = 1; k < mode; ++k) L *= s.dims[k];
    p.L = L;
  }
  if (!plan_digits(p, s)) return false;
  const int RT = stream_rt(s.R, op), RG = stream_rg(s.R, op);
  const int WSTR = (s.R % 2 == 0) ? s.R + 2 : s.R + 1;
  p.RS = s.R + (s.R & 1);
  // stage size: tools/sweep*.sh (DFMA consumers), tools/plan_sweep.py (MMA: 2 stages of ~52 KB)
  int stage_target = knob("CP_STAGE_BYTES", plan_mma_ok(p, s, op) ? 53248 : 40960);
  int cps, cpt = 1;
  if (plan_mma(p, s, op)) {
    // whole-column row blocks loaded by one tensor-map TMA per stage (launch_stream): 3 stages
    // of ~26 KB beat 2 of ~52 KB (c4b MTTKRP 0.153 -> 0.143 ms; tools/sweep_c4b.sh)
    if (tmap_geometry_ok(p) && path_flag("CP_STREAM_TMAP", 1)) stage_target = knob("CP_STAGE_BYTES", 26624);
    // stage: a multiple of 4 KS columns (k-steps of every k-group)
    const int unit = 4 * p.ks;
    cps = stage_target / (p.zcs * 8);
    cps = (cps / unit) * unit;
    if (cps < unit) cps = unit;
    if (cps > 64) cps = 64;
    p.zst = cps * p.zcs;
    // B fragments straight from the staged factor rows, times the slow digits' rows (also
    // staged): no weight warp whenever digit 0 is a factor mode
    const bool has_f0 = (p.ord[0] != p.mode);
    bool slow = false;
    for (int j = 1; j < p.nd; ++j)
      if (p.ord[j] != p.mode) slow = true;
    p.direct_w = has_f0 ? 1 : 0;
    p.srows = (has_f0 && slow && knob("CP_MMA_SROWS", 1)) ? 1 : 0;
    if (has_f0 && slow && !p.srows) p.direct_w = 0;
    // (cp_mttkrp) factor rows straight from the caller's column-major factors (tensor maps)
    if (fcm && op == OP_MTTKRP && p.direct_w) p.fcm = 1;
    const int RP = 8 * p.nt;
    if (op == OP_YL) p.red_doubles = (p.ks - 1) * p.Wmax * RP + 8;
    else if (p.mode != 0) p.red_doubles = kConsumerWarps * RP + 8;
    else p.red_doubles = 8;
  } else {
    // rows per consumer thread: the largest V dividing I1 with V * RT <= 32 accumulators, which
    // keeps the kernel at <= 96 registers and 2 CTAs/SM; residual pass: V <= 4 and V * R <= 64
    const int vmax_env = knob("CP_MAX_V", 8);
    const int vr_max = knob("CP_MAX_VR", 32);
    p.V = 1;
    for (int v : {8, 4, 2}) {
      if (v > vmax_env || p.I1 % v != 0) continue;
      if (op != OP_RESID && v * RT > vr_max && v > 2) continue;
      if (op == OP_RESID && (v > 4 || v * s.R > 64)) continue;
      p.V = v;
      break;
    }
    int maxW = (kConsumers / RG) * p.V;  // one column per sub-tile at most
    if (maxW > kMaxRows) maxW = kMaxRows;
    // row-block width: mode 0 MTTKRP uses narrower blocks (fewer column groups -> smaller I1 x R
    // partials); every other pass keeps whole columns in one CTA.
    int64_t Wt = p.I1;
    if (op != OP_RESID && p.mode == 0) {
      const int w0 = knob("CP_MTTKRP_W0", 512);
      if (p.I1 >= 2 * w0) Wt = w0;
    }
    if (op == OP_YL) {
      const int w0 = knob("CP_YL_W", 512);
      if (p.I1 >= 2 * w0) Wt = w0;
    }
    if (Wt > maxW) Wt = maxW;
    p.RB = (int)ceil_div(p.I1, Wt);
    int64_t W = ceil_div(p.I1, p.RB);
    while (W % p.V) ++W;
    p.Wmax = (int)W;
    const int U = p.Wmax / p.V;
    cpt = (kConsumers / (U * RG)) > 0 ? (kConsumers / (U * RG)) : 1;
    cps = stage_target / (p.Wmax * 8);
    if (cps < 1) cps = 1;
    if (cps >= cpt) cps = (cps / cpt) * cpt;
    else cps = cpt;
    if (cps > 64) cps = 64;
    p.zst = cps * p.Wmax;
    // consumers' shared reduction area (stream_kernel.cuh): residual pass: one double per warp;
    // mode >= 1 MTTKRP: one RT-vector per warp when every warp holds a single rank group (RG = 1
    // or U a multiple of 32 in every row block), else one per thread; Y_L pass with several
    // column slots: G regions of Wmax x R (G <= cpt - 1, within the generic budget); mode-0
    // MTTKRP reduces through the Z ring instead.
    const int generic = 256 * RT + 8;
    int red = 8;
    if (op == OP_MTTKRP && p.mode != 0) {
      const int64_t Wlast = p.I1 - (int64_t)(p.RB - 1) * p.Wmax;
      const bool warp_uniform = (RG == 1) || ((p.Wmax / p.V) % 32 == 0 && (Wlast / p.V) % 32 == 0);
      red = warp_uniform ? kConsumerWarps * RT + 8 : generic;
    } else if (op == OP_YL && cpt > 1) {
      int G = generic / (p.Wmax * s.R);
      if (G > cpt - 1) G = cpt - 1;
      if (G < 1) G = 1;
      red = G * p.Wmax * s.R;
    }
    p.red_doubles = red;
  }
  if (cps > p.Q) cps = (int)p.Q;
  p.cps = cps;
  p.zst = cps * (p.mma ? p.zcs : p.Wmax);
  if (p.mma) {
    // staged factor rows keep the At stride (one bulk copy per stage) and the weight rows the
    // DFMA kernel's stride.  Padding either to 8 (mod 16) doubles removes the B-fragment bank
    // conflicts but measured slower (per-row copies; smaller stages): CP_MMA_PAD_A/_W
    int st = p.RS;
    while (st % 16 != 8) ++st;
    p.ars = knob("CP_MMA_PAD_A", 0) ? st : p.RS;
    if (op == OP_RESID && p.direct_w && knob("CP_RESID_PAD_A", 1)) {
      // residual pass: B fragments read factor row gq, rank 4 kk + tq -- a row stride of 4
      // (mod 16) doubles spreads a half-warp over 16 bank pairs (one bulk copy per row)
      int sa = p.RS;
      while (sa % 16 != 4) ++sa;
      p.ars = sa;
    }
    p.wstr = knob("CP_MMA_PAD_W", 0) ? st : WSTR;
    if (p.direct_w && knob("CP_MMA_WSTR0", 1)) p.wstr = 0;  // no weight rows
    if (p.fcm) {
      p.ars = 0;
      p.wstr = 0;
    }
  } else {
    p.ars = p.RS;
    p.wstr = WSTR;
  }
  // ring: CP_RING_BYTES (default 96 KB) of stages, at least 2; the MMA kernels also keep the whole
  // CTA within the 2-CTAs/SM shared-memory budget (113 KB) by shrinking the stage if needed
  const int cap = knob("CP_SMEM_CAP", 113 * 1024);
  p.gjsm = (p.mma && p.direct_w) ? gamma_job_smem_doubles(s.R) : 0;  // Gamma job (gamma_job.cuh)
  const int unit = p.mma ? 4 * p.ks : 1;
  int stage_doubles = 0, nst = 2;
  // staged factor rows per stage (abuf) and slow-row slots (sbuf); fcm: the rank-major box
  // [R][fs], fs = 4 (mod 16) doubles >= cps, slots padded to 128 B (TMA destinations)
  auto stage_bufs = [&]() {
    if (p.fcm) {
      p.fs = cps + 1;  // (+1: the box starts at an even row, TMA coordinates are 16-B aligned)
      while (p.fs % 16 != 4) ++p.fs;
      p.astage = (int)(ceil_div((int64_t)s.R * p.fs, 16) * 16);
      p.srs = (int)(ceil_div(2 * (int64_t)s.R, 16) * 16);
      p.sstr = 2;
    } else {
      p.fs = 0;
      p.astage = cps * p.ars;
      p.srs = p.RS;
      p.sstr = 1;
    }
  };
  for (;;) {
    stage_bufs();
    stage_doubles = p.zst + p.astage + cps * p.wstr + (p.srows ? kMaxDigits * p.srs : 0);
    nst = knob("CP_RING_BYTES", 96 * 1024) / (stage_doubles * 8);
    if (nst < 2) nst = 2;
    if (nst > 8) nst = 8;
    // mode-0 slot / k-group reduction reuses the Z ring: it must hold the reduced blocks
    const int64_t need = p.mma ? (int64_t)(p.ks - 1) * p.Wmax * 8 * p.nt : (int64_t)p.Wmax * s.R;
    while ((int64_t)nst * p.zst < need) ++nst;
    const int bytes = (nst * stage_doubles + p.red_doubles + p.gjsm + 32) * 8 + nst * 88 + 64;
    if (!p.mma || bytes <= cap || cps <= unit) break;
    cps -= unit;
    p.cps = cps;
    p.zst = cps * p.zcs;
  }
  stage_bufs();
  p.nstages = nst;
  p.dbg = knob("CP_STREAM_DBG", 0);
  p.keep_q = 0;
  p.smem_bytes = (nst * stage_doubles + p.red_doubles + p.gjsm + 32) * 8 + nst * 88 + 64;
  if (p.smem_bytes > 200 * 1024) return false;
  const int occ = p.mma ? stream_mma_occupancy(p.nt, p.mt, op, p.smem_bytes)
                        : stream_occupancy(s.R, p.V, op, p.smem_bytes);
  const int ctas = knob("CP_CTAS_PER_SM", 0);
  const int64_t Gtot = (int64_t)num_sms * (ctas > 0 ? (ctas < occ ? ctas : occ) : occ);
  int64_t Gc = Gtot / p.RB;
  if (Gc < 1) Gc = 1;
  const int64_t maxGc = ceil_div(p.Q, cps);
  if (Gc > maxGc) Gc = maxGc;
  if (Gc > p.Q) Gc = p.Q;
  p.Gc = (int)Gc;
  if (p.mode == 0) {
    p.slots = 1;
  } else {
    const int64_t maxrange = ceil_div(p.Q, Gc);
    p.slots = (int)(maxrange / p.Qn + 2);
  }
  return true;
}

size_t stream_part_doubles(const StreamPlan &p) {
  if (p.op == OP_RESID) return (size_t)p.Gc * p.RB;
  if (p.mode == 0) return (size_t)p.Gc * p.I1 * p.R;
  return (size_t)p.Gc * p.RB * p.slots * p.R;
}

// ---------------------------------------------------------------- live kernel timing
constexpr int kProfMax = 8192;
static bool g_prof_on = false;
static int g_prof_n = 0;
static cudaEvent_t g_prof_ev[2 * kProfMax];
static double g_prof_bytes[kProfMax];
static bool g_prof_init = false;

static double stream_alg_bytes(const StreamPlan &p) {
  double P = 1.0, fac = 0.0;
  for (int k = 0; k < p.N; ++k) {
    P *= (double)p.dims[k];
    if (k != p.mode || p.op == OP_RESID) fac += (double)p.dims[k] * p.R;
  }
  double out = (p.op == OP_RESID) ? 0.0 : (double)p.dims[p.mode] * p.R;
  if (p.op == OP_YL) out = (double)p.dims[0] * p.dims[1] * p.R;  // Y_L (I0 x I1 x R) written
  return 8.0 * (P + fac + out);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link)
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// The stage tensor map of an MMA plan (StreamPlan::use_tmap), when the plan qualifies: the row
// block is the whole column (RB = 1) and padded (zcs > Wb: the out-of-bounds box rows fill the
// padding with zeros), 16-byte row strides, box within the TMA limits (<= 256 per dimension).
static bool encode_stage_tmap(StreamPlan &p) {
  if (!tmap_geometry_ok(p) || p.cps > 256) return false;
  const int64_t qs = p.qsd[0];
  if (qs < 1 || p.Q % qs != 0 || p.Q / qs > 0x7fffffffLL || qs > 0x7fffffffLL) return false;  // (int32 TMA coordinates)
  if ((p.zst * 8) % 128 != 0) return false;  // stage slots must stay 128-B aligned
  auto enc = tmap_encoder();
  if (enc == nullptr) return false;
  const cuuint64_t gdim[3] = {(cuuint64_t)p.I1, (cuuint64_t)qs, (cuuint64_t)(p.Q / qs)};
  const cuuint64_t gstride[2] = {(cuuint64_t)p.I1 * 8, (cuuint64_t)(p.I1 * qs * 8)};
  const cuuint32_t box[3] = {(cuuint32_t)p.zcs, 1u, (cuuint32_t)p.cps};
  const cuuint32_t estride[3] = {1u, 1u, 1u};
  const CUresult r = enc(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(p.Z), gdim, gstride, box,
                         estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// The factor tensor maps of an fcm plan (StreamPlan::fcm): 2-D views {I_k, R} of the caller's
// column-major factors (row stride I_k * 8 bytes, a multiple of 16: I_k even, 16-B aligned base;
// fcm_ok() checks before the plan is chosen).  fmap[0]: box {fs, R} of A^(ord[0]); fmap[j]:
// box {2, R} of the slow digit j's factor (TMA box rows must be 16-byte multiples).
static bool encode_factor_maps(StreamPlan &p) {
  auto enc = tmap_encoder();
  if (enc == nullptr) return false;
  auto one = [&](CUtensorMap *m, int k, unsigned box0) -> bool {
    const int64_t I = p.dims[k];
    if ((I & 1) || ((uintptr_t)p.Af[k] % 16) != 0 || I > 0x7fffffffLL) return false;
    const cuuint64_t gdim[2] = {(cuuint64_t)I, (cuuint64_t)p.R};
    const cuuint64_t gstride[1] = {(cuuint64_t)I * 8};
    const cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)p.R};
    const cuuint32_t es[2] = {1u, 1u};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(p.Af[k]), gdim, gstride, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
  };
  if (!one(&p.fmap[0], p.ord[0], (unsigned)p.fs)) return false;
  for (int j = 1; j < p.nd; ++j)
    if (p.ord[j] != p.mode && !one(&p.fmap[j], p.ord[j], 2u)) return false;
  return true;
}

// the caller's factors can be staged through tensor maps (every factor mode of the plan)
static bool fcm_ok(const StreamPlan &p, const cp_shape &s, const double *const *A) {
  for (int k = 0; k < s.N; ++k) {
    if (k == p.mode) continue;
    if ((s.dims[k] & 1) || A[k] == nullptr || ((uintptr_t)A[k] % 16) != 0) return false;
  }
  return true;
}

cudaError_t launch_stream(const StreamPlan &p0, cudaStream_t st) {
  StreamPlan p = p0;
  {
    // L2 residency across passes (DESIGN 6.8): for a tensor well beyond L2, the first
    // CP_L2KEEP_MB MiB of Z (default 40) are fetched evict_last and the rest evict_first, so
    // consecutive passes over the same Z re-read that slice from L2
    const int64_t keep_mb = knob("CP_L2KEEP_MB", 40);
    double P = 1.0;
    for (int k = 0; k < p.N; ++k) P *= (double)p.dims[k];
    if (keep_mb > 0 && p.V >= 2 && 8.0 * P >= 96.0 * (1 << 20)) p.keep_q = (keep_mb << 20) / (8 * p.I1);
  }
  p.use_tmap = 0;
  if (p.mma && path_flag("CP_STREAM_TMAP", 1)) p.use_tmap = encode_stage_tmap(p) ? 1 : 0;
  if (p.fcm && !encode_factor_maps(p)) return cudaErrorInvalidValue;
  const StreamEntry &e = p.mma ? stream_mma_entry(p.nt, p.mt, p.op, stream_mma_feat(p) || path_flag("CP_STREAM_LEAN", 1) == 0)
                              : stream_entry(p.R, p.V, p.op);
  ++g_launches;
  const bool prof = g_prof_on && g_prof_n < kProfMax;
  if (prof) cudaEventRecord(g_prof_ev[2 * g_prof_n], st);
  const cudaError_t err = e.launch(p, st);
  if (prof) {
    cudaEventRecord(g_prof_ev[2 * g_prof_n + 1], st);
    g_prof_bytes[g_prof_n] = stream_alg_bytes(p);
    ++g_prof_n;
  }
  return err;
}

// ---------------------------------------------------------------- workspace layout
struct Layout {
  size_t status, Ups, gpart0, gpart1, dotM, dotF, gradp, normp, residp, part, At[CP_MAX_N], total;
  int gp_max, grad_max, norm_blocks, prep_blocks;
  size_t gpre;
  int rpc[CP_MAX_N], sp[CP_MAX_N];  // row blocking of the solve / gradient / reduce kernels
  int nsolve[CP_MAX_N], ngrad[CP_MAX_N];
  StreamPlan plans[CP_MAX_N];
  StreamPlan gplans[CP_MAX_N];  // cp_mttkrp: column-major-factor (fcm) variants of the MMA plans
  StreamPlan resid;
  // dimension-tree sweep (N >= 3): pass 1 = OP_YL over Z (mode-1 segments), pass 2 = mode-2
  // MTTKRP of Z viewed as I0 x I1 x J (J = prod_{k>=2} I_k)
  bool tree;
  StreamPlan yl_plan, p2_plan;
  cp_shape s3;
  int rpc2, sp2, nyr;
  size_t yl, edge, mbuf, yr, segtab, m0part, linv;
  size_t tick;  // tagged completion words (StreamPlan::tick): 3 + max I_n
  size_t rowdot;  // TailSolve: per-row <M,A>, <F,A> of the last mode (2 x max I_n)
  size_t tailtick;  // TailSolve: u32 words (max I_n segment tickets, grid ticket, Gamma-job flag),
                    // right after segtab: the prep kernel zeroes both in one range
  int64_t maxI;
  size_t ntmp;  // cp_als_sweeps with CP_SWEEPS_NORMALIZE: normalization scratch (sum_n I_n R)
};

static size_t align_up(size_t x) { return (x + 31) & ~(size_t)31; }  // 256 B in doubles

static bool make_layout(Layout &L, const cp_shape &s) {
  memset(&L, 0, sizeof(L));
  const int sms = device_sms();
  const int R = s.R;
  size_t part = 0;
  int64_t maxI = 1;
  for (int n = 0; n < s.N; ++n) {
    if (!make_stream_plan(L.plans[n], s, n, OP_MTTKRP, sms)) return false;
    size_t d = stream_part_doubles(L.plans[n]);
    if (d > part) part = d;
    if (!L.plans[n].mma || !make_stream_plan(L.gplans[n], s, n, OP_MTTKRP, sms, true) || !L.gplans[n].fcm)
      L.gplans[n].mma = 0;
    if (L.gplans[n].mma && (d = stream_part_doubles(L.gplans[n])) > part) part = d;
    row_blocking(L.plans[n], &L.rpc[n], &L.sp[n]);
    L.nsolve[n] = (int)ceil_div(s.dims[n], L.rpc[n]);
    if (L.nsolve[n] > L.gp_max) L.gp_max = L.nsolve[n];
    L.ngrad[n] = L.nsolve[n];
    if (L.ngrad[n] > L.grad_max) L.grad_max = L.ngrad[n];
    if (s.dims[n] > maxI) maxI = s.dims[n];
  }
  L.prep_blocks = 0;
  for (int k = 0; k < s.N; ++k) L.prep_blocks += (int)ceil_div(s.dims[k], kPrepRows);
  if (!make_stream_plan(L.resid, s, 0, OP_RESID, sms)) return false;
  L.tree = (s.N >= 3) && path_flag("CP_SWEEP_TREE", 1) != 0;
  if (L.tree) {
    if (!make_stream_plan(L.yl_plan, s, 1, OP_YL, sms)) return false;
    memset(&L.s3, 0, sizeof(L.s3));
    L.s3.N = 3;
    L.s3.R = R;
    L.s3.dims[0] = s.dims[0];
    L.s3.dims[1] = s.dims[1];
    L.s3.dims[2] = 1;
    for (int k = 2; k < s.N; ++k) L.s3.dims[2] *= s.dims[k];
    if (L.s3.dims[2] > 0x7fffffff || s.dims[0] * R > 0x7fffffff) L.tree = false;  // 32-bit Y_L block indices
  }
  if (L.tree) {
    if (!make_stream_plan(L.p2_plan, L.s3, 2, OP_MTTKRP, sms)) return false;
    const size_t d = stream_part_doubles(L.p2_plan);
    if (d > part) part = d;
    row_blocking(L.p2_plan, &L.rpc2, &L.sp2);
    {
      // the tree's mode-0 solve (ymm0 partials) and its direct-M solves (rpc 256 / R)
      int rpc0, sp0;
      ymm0_solve_blocking(R, s.dims[1], &rpc0, &sp0);
      const int n0 = (int)ceil_div(s.dims[0], rpc0);
      if (n0 > L.gp_max) L.gp_max = n0;
      const int rpcd = 256 / R > 0 ? 256 / R : 1;
      for (int k = 0; k < s.N; ++k) {
        const int nk = (int)ceil_div(s.dims[k], rpcd);
        if (nk > L.gp_max) L.gp_max = nk;
      }
      const int n2 = (int)ceil_div(s.dims[2], L.rpc2);
      if (n2 > L.gp_max) L.gp_max = n2;
      // the ylsolve kernels (modes 0, 1) write one Gram partial and one <F, A> per 8-CTA cluster
      for (int k = 0; k < 2; ++k) {
        const int nc = ylsolve_clusters(s.dims[k]);
        if (nc > L.gp_max) L.gp_max = nc;
      }
      if (L.gp_max > L.grad_max) L.grad_max = L.gp_max;  // cp_fit's gradient grids (same blocking)
    }
    L.nyr = (int)ceil_div(L.s3.dims[2], L.rpc2);
  }
  L.norm_blocks = 2 * sms;
  size_t off = 0;
  L.status = off; off = align_up(off + 8);
  L.Ups = off; off = align_up(off + (size_t)s.N * R * R);
  L.gpre = off; off = align_up(off + (size_t)L.prep_blocks * R * R);
  L.gpart0 = off; off = align_up(off + (size_t)L.gp_max * R * R);
  L.gpart1 = off; off = align_up(off + (size_t)L.gp_max * R * R);
  L.dotM = off; off = align_up(off + L.gp_max);
  L.dotF = off; off = align_up(off + (size_t)s.N * L.gp_max);
  L.gradp = off; off = align_up(off + (size_t)s.N * L.grad_max);
  L.normp = off; off = align_up(off + L.norm_blocks);
  L.residp = off; off = align_up(off + stream_part_doubles(L.resid));
  for (int k = 0; k < s.N; ++k) {
    L.At[k] = off;
    off = align_up(off + (size_t)s.dims[k] * (R + (R & 1)));
  }
  L.part = off; off = align_up(off + part);
  if (L.tree) {
    const StreamPlan &y = L.yl_plan;
    L.yl = off; off = align_up(off + (size_t)s.dims[0] * s.dims[1] * R);
    L.edge = off; off = align_up(off + (size_t)2 * y.Gc * y.RB * s.dims[0] * R);
    L.mbuf = off; off = align_up(off + (size_t)maxI * R);
    L.m0part = off; off = align_up(off + (size_t)32 * s.dims[0] * R);  // ymm0 range partials (<= 32)
    L.linv = off; off = align_up(off + (size_t)s.N * R * R);  // L^{-1} of every Gamma^(n)
    L.yr = off; off = align_up(off + (size_t)L.s3.dims[2] * R);
    L.segtab = off; off = align_up(off + (size_t)(s.dims[1] * y.RB + 1) / 2);  // u32 ticket per (segment, row block)
    L.tailtick = off; off = align_up(off + (size_t)(maxI + 2 + 1) / 2);
  }
  L.tick = off; off = align_up(off + 3 + (size_t)maxI);
  L.rowdot = off; off = align_up(off + 2 * (size_t)maxI);
  L.maxI = maxI;
  {
    size_t sumIR = 0;
    for (int k = 0; k < s.N; ++k) sumIR += (size_t)s.dims[k] * R;
    L.ntmp = off;
    off = align_up(off + sumIR);
  }
  L.total = off * sizeof(double);
  return true;
}

// Layouts (all launch plans of a shape) cached per (device, shape, planning path flags): planning
// costs ~10-20 us of host time per call, as much as a c3 pass on the device.  A small most-
// recently-used list; entries are immutable and shared.  Experiment builds (knobs from the
// environment may change between calls) always plan afresh.
static std::shared_ptr<const Layout> get_layout(const cp_shape &s) {
#ifdef CP_EXPERIMENTS
  auto fresh = std::make_shared<Layout>();
  if (!make_layout(*fresh, s)) return nullptr;
  return fresh;
#else
  struct Key {
    int dev, N, R, flags[4];
    int64_t dims[CP_MAX_N];
    bool operator==(const Key &o) const {
      if (dev != o.dev || N != o.N || R != o.R) return false;
      for (int i = 0; i < 4; ++i)
        if (flags[i] != o.flags[i]) return false;
      for (int k = 0; k < N; ++k)
        if (dims[k] != o.dims[k]) return false;
      return true;
    }
  };
  Key key;
  memset(&key, 0, sizeof(key));
  key.dev = current_device();
  key.N = s.N;
  key.R = s.R;
  for (int k = 0; k < s.N && k < CP_MAX_N; ++k) key.dims[k] = s.dims[k];
  key.flags[0] = path_flag("CP_STREAM_MMA", 1);
  key.flags[1] = path_flag("CP_RESID_MMA", 1);
  key.flags[2] = path_flag("CP_STREAM_TMAP", 1);
  key.flags[3] = path_flag("CP_SWEEP_TREE", 1);
  static std::mutex mu;
  static std::vector<std::pair<Key, std::shared_ptr<const Layout>>> cache;  // most recent first
  constexpr size_t kMaxLayouts = 32;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (size_t i = 0; i < cache.size(); ++i) {
      if (cache[i].first == key) {
        auto hit = cache[i];
        cache.erase(cache.begin() + (long)i);
        cache.insert(cache.begin(), hit);
        return hit.second;
      }
    }
  }
  auto fresh = std::make_shared<Layout>();
  if (!make_layout(*fresh, s)) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  cache.insert(cache.begin(), {key, fresh});
  if (cache.size() > kMaxLayouts) cache.pop_back();
  return fresh;
#endif
}

// Arguments of the prep kernel (At copies of every factor except skip_mode; per-block partial
// Grams when grams) and where its Gram partials land.
static void fill_prep(const cp_shape &s, const Layout &L, double *w, const double *const *A,
                      int skip_mode, bool grams, double *status, PrepArgs &pa, PrepGrams &pg) {
  memset(&pa, 0, sizeof(pa));
  memset(&pg, 0, sizeof(pg));
  pa.N = s.N;
  pa.R = s.R;
  for (int k = 0; k < s.N; ++k) {
    pa.dims[k] = s.dims[k];
    pa.A[k] = (k == skip_mode) ? nullptr : A[k];
    pa.At[k] = w + L.At[k];
  }
  pa.gpre = grams ? w + L.gpre : nullptr;
  pa.status = status;
  prep_blocks(s, pa, pg);
  pg.gpre = w + L.gpre;
}

static int check_shape(const cp_shape *s, int minN) {
  if (s == nullptr) return CP_EINVAL;
  if (s->N < minN || s->N > CP_MAX_N || s->R < 1 || s->R > CP_MAX_R) return CP_EINVAL;
  double P = 1.0;
  for (int k = 0; k < s->N; ++k) {
    if (s->dims[k] < 1) return CP_EDIM;
    P *= (double)s->dims[k];
  }
  if (P >= 1125899906842624.0) return CP_EDIM;  // 2^50 elements
  return CP_OK;
}

static bool aligned(const void *p, size_t a) { return ((uintptr_t)p % a) == 0; }

static int check_ws(const Layout &L, void *ws, size_t ws_bytes) {
  if (ws == nullptr || !aligned(ws, 256)) return CP_EINVAL;
  if (ws_bytes < L.total) return CP_EWORKSPACE;
  return CP_OK;
}

static int ret_cuda(cudaError_t e) { return e == cudaSuccess ? CP_OK : CP_ECUDA; }

}  // namespace cpk

using namespace cpk;

extern "C" {

size_t cp_workspace_bytes(const cp_shape *s) {
  if (check_shape(s, 1) != CP_OK) return 0;
  if (s->N < 2) {
    // cp_norm2 only needs its block partials
    return (size_t)(2 * device_sms() + 64) * sizeof(double);
  }
  const auto Lp = get_layout(*s);
  return Lp ? Lp->total : 0;
}

int cp_norm2(const cp_shape *s, const double *Z, double *out, void *ws, size_t ws_bytes,
             cp_stream_t stream) {
  g_launches = 0;
  int st = check_shape(s, 1);
  if (st) return st;
  if (!Z || !out || !aligned(Z, 16)) return CP_EINVAL;
  const size_t need = cp_workspace_bytes(s);
  if (ws == nullptr || !aligned(ws, 256)) return CP_EINVAL;
  if (ws_bytes < need) return CP_EWORKSPACE;
  int64_t P = 1;
  for (int k = 0; k < s->N; ++k) P *= s->dims[k];
  const int nb = 2 * device_sms();
  double *part = static_cast<double *>(ws);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (launch_k(norm2_kernel, dim3(nb), dim3(512), 0, cs, Z, P, part) != cudaSuccess) return CP_ECUDA;
  if (launch_k(norm2_final_kernel, dim3(1), dim3(256), 0, cs, (const double *)part, nb, out) != cudaSuccess) return CP_ECUDA;
  g_launches = 2;
  return CP_OK;
}

int cp_mttkrp(const cp_shape *s, const double *Z, const double *const *A, int32_t mode, double *M,
              void *ws, size_t ws_bytes, cp_stream_t stream) {
  g_launches = 0;
  int st = check_shape(s, 2);
  if (st) return st;
  if (!Z || !A || !M || mode < 0 || mode >= s->N || !aligned(Z, 16)) return CP_EINVAL;
  for (int k = 0; k < s->N; ++k)
    if (k != mode && A[k] == nullptr) return CP_EINVAL;
  const auto Lp = get_layout(*s);
  if (!Lp) return CP_EINVAL;
  const Layout &L = *Lp;
  if ((st = check_ws(L, ws, ws_bytes))) return st;
  double *w = static_cast<double *>(ws);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  int nl = 2;
  StreamPlan p;
  // 0: never, 1: modes >= 1, 2: every mode (default; r02: mode 0 c3 43.0 -> 40.9 us, c4b
  // 162.5 -> 150.0 us against prep + At copies, tools/mttkrp_ab.py)
  const int fcm_sel = path_flag("CP_MTTKRP_FCM", 2);
  if ((mode != 0 || fcm_sel >= 2) && fcm_sel > 0 && L.gplans[mode].mma && fcm_ok(L.gplans[mode], *s, A)) {
    // MMA plans: the producer stages the factor rows from the caller's column-major factors
    // through tensor maps -- no prep launch
    p = L.gplans[mode];
    for (int k = 0; k < s->N; ++k) p.Af[k] = A[k];
  } else {
    PrepArgs pa;
    PrepGrams pg;
    fill_prep(*s, L, w, A, mode, false, nullptr, pa, pg);
    if (launch_prep(pa, cs) != cudaSuccess) return CP_ECUDA;
    p = L.plans[mode];
    for (int k = 0; k < s->N; ++k) p.At[k] = w + L.At[k];
    nl = 3;
  }
  p.Z = Z;
  p.part = w + L.part;
  // MMA plans finish M inside the pass: no reduce launch.  CP_MTTKRP_FUSED = 1 (default): modes
  // >= 1 when a CTA touches few segments (tagged tickets, one round trip per 32 segments at the
  // CTA's end); 2: also mode 0 (grid barrier + sliced sum; measured slower than the separate
  // reduce: c3 27.6 -> 34.8 us, c4a 199 -> 206 us per call).
  const int fused = path_flag("CP_MTTKRP_FUSED", 1);
  if (p.mma && fused > 0 && (mode == 0 ? fused >= 2 : p.slots <= 32)) {
    p.Mout = M;
    p.tick = reinterpret_cast<unsigned long long *>(w + L.tick);
    p.tag = next_tag();
    if (launch_stream(p, cs) != cudaSuccess) return CP_ECUDA;
    g_launches = nl - 1;
    return CP_OK;
  }
  if (launch_stream(p, cs) != cudaSuccess) return CP_ECUDA;
  const ReduceGeom g = reduce_geom(p);
  if (g.mode0 && !g.direct && knob("CP_REDUCE0_COALESCED", 1)) {
    const int64_t S = g.In_rows * g.R;
    if (launch_kc(kPdlWide, reduce_mode0_kernel, dim3((unsigned)ceil_div(S, 32)), dim3(1024), 0, cs,
                  (const double *)g.part, g.Gc, S, M) != cudaSuccess)
      return CP_ECUDA;
  } else if (launch_k(reduce_mttkrp_kernel, dim3(L.nsolve[mode]), dim3(256), 0, cs, g, L.rpc[mode], L.sp[mode], M) !=
             cudaSuccess) {
    return CP_ECUDA;
  }
  g_launches = nl;
  return CP_OK;
}

// small tensors (coarse multigrid levels): the fused shared-memory sweep kernel (small_sweep.cu)
static bool use_small_sweep(const cp_shape &s) {
  return path_flag("CP_SMALL_SWEEP", 1) != 0 && small_sweep_smem_bytes(s) != 0 &&
         small_sweep_smem_bytes(s) <= (size_t)knob("CP_SMALL_SWEEP_SMEM", 200 * 1024);
}

static int sweep_impl(const cp_shape *s, const double *Z, const double *normZ2, double *const *A,
                      const double *const *F, double *out, void *ws, size_t ws_bytes, cp_stream_t stream,
                      bool first, bool steady, bool defer_ok = false, bool prev_deferred = false,
                      bool *deferred = nullptr);

int cp_als_sweep(const cp_shape *s, const double *Z, const double *normZ2, double *const *A,
                 const double *const *F, double *out, void *ws, size_t ws_bytes,
                 cp_stream_t stream) {
  return cp_als_sweeps(s, Z, normZ2, A, F, 1, 0, out, ws, ws_bytes, stream);
}

int cp_als_sweeps(const cp_shape *s, const double *Z, const double *normZ2, double *const *A,
                  const double *const *F, int32_t nsweeps, int32_t flags, double *out, void *ws,
                  size_t ws_bytes, cp_stream_t stream) {
  g_launches = 0;
  int st = check_shape(s, 2);
  if (st) return st;
  if (!Z || !normZ2 || !A || !out || !aligned(Z, 16) || nsweeps < 1 || (flags & ~CP_SWEEPS_NORMALIZE))
    return CP_EINVAL;
  const bool norm = (flags & CP_SWEEPS_NORMALIZE) != 0;
  for (int k = 0; k < s->N; ++k)
    if (A[k] == nullptr) return CP_EINVAL;
  const auto Lp = get_layout(*s);
  if (!Lp) return CP_EINVAL;
  const Layout &L = *Lp;
  if ((st = check_ws(L, ws, ws_bytes))) return st;
  if (use_small_sweep(*s) && path_flag("CP_TINY_SWEEP", 1) != 0 && tiny_sweep_ok(*s)) {
    // the tiniest levels (P <= 512, R <= 4): one warp runs the whole call (tiny_sweep.cu)
    if (launch_tiny_sweep(*s, Z, normZ2, A, F, nsweeps, out, reinterpret_cast<cudaStream_t>(stream), norm) !=
        cudaSuccess)
      return CP_ECUDA;
    g_launches = 1;
    return CP_OK;
  }
  if (use_small_sweep(*s)) {
    if (launch_small_sweep(*s, Z, normZ2, A, F, nsweeps, out, reinterpret_cast<cudaStream_t>(stream), nullptr,
                           false, norm) != cudaSuccess)
      return CP_ECUDA;
    g_launches = 1;
    return CP_OK;
  }
  int total = 0;
  bool deferred = false;
  for (int k = 0; k < nsweeps; ++k) {
    // sweeps k >= 1 without normalization in between run steady-state: the previous sweep's
    // solves left every At copy and Gram total current, so no prep launch; a sweep that is not the
    // call's last may solve its last mode inside the pass and leave Upsilon^(N-1) to the next
    // sweep's Gamma^(0) job (TailSolve; its f is not needed: the call returns the last sweep's)
    const bool prev = deferred;
    if ((st = sweep_impl(s, Z, normZ2, A, F, out, ws, ws_bytes, stream, k == 0, k > 0 && !norm,
                         k + 1 < nsweeps && !norm, prev, &deferred)))
      return st;
    total += g_launches;
    if (norm) {  // cp_normalize_sort(sort = 0) with the sweep workspace's own scratch region
      NormArgs na;
      memset(&na, 0, sizeof(na));
      na.N = s->N;
      na.R = s->R;
      int64_t o = 0;
      for (int n = 0; n < s->N; ++n) {
        na.dims[n] = s->dims[n];
        na.A[n] = A[n];
        na.off[n] = o;
        o += s->dims[n] * s->R;
      }
      na.tmp = static_cast<double *>(ws) + L.ntmp;
      if (launch_normalize_sort(na, reinterpret_cast<cudaStream_t>(stream)) != cudaSuccess) return CP_ECUDA;
      ++total;
    }
  }
  g_launches = total;
  return CP_OK;
}

// One sweep of the general path.  first = false: a later sweep of the same cp_als_sweeps call --
// the status word is not reset, so a failure in an earlier sweep stays reported and every later
// solve skips (the fused small kernel likewise stops at the first failure).  steady: the factors
// are unchanged since the previous sweep of this call (no normalization in between), whose solves
// wrote the row-major copies At and the Gram totals Ups of every mode -- the prep launch (At
// copies + partial Grams) is skipped and every Gram of a not-yet-updated factor is read as a total
// (bitwise the same as the previous sweep's totals; the tickets were reset by their last users).
// defer_ok: another steady sweep of the same call follows; prev_deferred: the previous sweep left
// Upsilon^(2) to this sweep's Gamma^(0) job; *deferred: this sweep did so.
static int sweep_impl(const cp_shape *s, const double *Z, const double *normZ2, double *const *A,
                      const double *const *F, double *out, void *ws, size_t ws_bytes, cp_stream_t stream,
                      bool first, bool steady, bool defer_ok, bool prev_deferred, bool *deferred) {
  g_launches = 0;
  if (deferred != nullptr) *deferred = false;
  int st;
  const auto Lp = get_layout(*s);
  if (!Lp) return CP_EINVAL;
  const Layout &L = *Lp;
  double *w = static_cast<double *>(ws);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  const int N = s->N, R = s->R;

  PrepArgs pa;
  PrepGrams pg;
  fill_prep(*s, L, w, (const double *const *)A, -1, true, w + L.status, pa, pg);
  pa.keep_status = first ? 0 : 1;
  const bool yl_inline = L.tree && L.yl_plan.mma && knob("CP_YL_INLINE_FIX", 1);
  if (L.tree) {
    // u32 completion words zeroed by prep: the Y_L segment tickets (stream_mma.cuh
    // yl_complete_segment) and, contiguous after them, the tail solve's words (sweep_tail)
    const size_t z0 = yl_inline ? L.segtab : L.tailtick;
    pa.zero = reinterpret_cast<unsigned *>(w + z0);
    pa.nzero = (int)((L.tailtick - z0) * 2 + (size_t)L.maxI + 2);
  }
  // experiments only (-DCP_EXPERIMENTS builds): CP_SWEEP_SKIP bitmask drops launches (timing of
  // the rest; results wrong).  Always 0 in the shipped library.
  const int skip = knob("CP_SWEEP_SKIP", 0);
  int launches = 0;
  if (steady) {
    pg.tot = w + L.Ups;
  } else {
    if (!(skip & 1) && launch_prep(pa, cs) != cudaSuccess) return CP_ECUDA;
    launches = 1;
  }
  double *gp[2] = {w + L.gpart0, w + L.gpart1};
  int grid_of[CP_MAX_N] = {0};
  // a4 for mode n from M given by rg (stream partials or a plain M buffer)
  auto solve_mode = [&](int n, const ReduceGeom &rg, int rpc, int sp, const double *linv = nullptr) -> bool {
    SolveArgs sa;
    memset(&sa, 0, sizeof(sa));
    sa.N = N;
    sa.R = R;
    sa.mode = n;
    sa.prev_mode = n - 1;
    sa.nprev = (n > 0) ? grid_of[n - 1] : 0;
    sa.rpc = rpc;
    sa.sp = sp;
    sa.In = s->dims[n];
    sa.rg = rg;
    sa.pg = pg;
    sa.F = (F != nullptr) ? F[n] : nullptr;
    sa.A = A[n];
    sa.At = w + L.At[n];
    sa.Ups = w + L.Ups;
    sa.gprev = (n > 0) ? gp[(n - 1) & 1] : nullptr;
    sa.gcur = gp[n & 1];
    sa.dotM = w + L.dotM;
    sa.dotF = w + L.dotF + (size_t)n * L.gp_max;
    sa.status = w + L.status;
    sa.dbg = knob("CP_SOLVE_DBG", 0);
    sa.linv = linv;
    grid_of[n] = (int)ceil_div(s->dims[n], rpc);
    if (n == N - 1) {
      // the sweep's last solve also evaluates f, f~ (finalize_body in its last block)
      sa.fin_on = 1;
      sa.ticket = reinterpret_cast<unsigned *>(w + L.status + kTicketSlot);
      FinalizeArgs &fa = sa.fin;
      fa.N = N;
      fa.R = R;
      fa.nlast = grid_of[N - 1];
      fa.dot_stride = L.gp_max;
      for (int k = 0; k < N; ++k) fa.nsolve[k] = grid_of[k];
      fa.glast = gp[(N - 1) & 1];
      fa.dotM_last = w + L.dotM;
      fa.dotF = w + L.dotF;
      fa.Ups = w + L.Ups;
      fa.normZ2 = normZ2;
      fa.status = w + L.status;
      fa.out = out;
    }
    ++launches;
    if (skip & (4 << n)) return true;
    return launch_solve(sa, grid_of[n], cs) == cudaSuccess;
  };
  const int RS = R + (R & 1);
  const int rpc_d = 256 / R > 0 ? 256 / R : 1;
  const int RR = R * R;
  // Gamma^(n) job (gamma_job.cuh): Upsilon^(k) for k > n from the prep partials (old factors),
  // k = n-1 from the previous solve's partials, k < n-1 from the totals earlier jobs wrote
  const bool jobs = L.tree && knob("CP_GAMMA_JOBS", 1) != 0;
  auto gamma_job = [&](int n) -> GammaJob {
    GammaJob g;
    memset(&g, 0, sizeof(g));
    g.on = 1;
    g.N = N;
    g.R = R;
    g.mode = n;
    for (int k = 0; k < N; ++k) {
      if (k == n) continue;
      if (k > n && steady) {
        g.src[k] = w + L.Ups + (size_t)k * RR;
        g.cnt[k] = 0;
      } else if (k > n) {
        g.src[k] = w + L.gpre + (size_t)pg.blk_off[k] * RR;
        g.cnt[k] = pg.nblk[k];
      } else if (k == n - 1) {
        g.src[k] = gp[k & 1];
        g.cnt[k] = grid_of[k];
      } else {
        g.src[k] = w + L.Ups + (size_t)k * RR;
        g.cnt[k] = 0;
      }
    }
    g.ups = w + L.Ups;
    g.linv = w + L.linv + (size_t)n * RR;
    g.status = w + L.status;
    if (n == 0 && prev_deferred) {
      // the previous sweep's in-pass tail solve wrote the rows of At^(2) only
      g.gram_mode = 2;
      g.gram_RS = RS;
      g.gram_rows = s->dims[2];
      g.gram_At = w + L.At[2];
    }
    return g;
  };
  if (L.tree) {
    // ---- dimension-tree sweep: two passes over Z instead of N ----
    StreamPlan p1 = L.yl_plan;
    p1.Z = Z;
    for (int k = 0; k < N; ++k) p1.At[k] = w + L.At[k];
    p1.yl = w + L.yl;
    p1.edge = w + L.edge;
    p1.segcnt = yl_inline ? reinterpret_cast<unsigned *>(w + L.segtab) : nullptr;
    p1.part = nullptr;
    // Gamma^(0) (Grams of the old factors only) rides in the Y_L pass's idle weight warp
    const bool job0 = jobs && p1.mma && p1.direct_w;
    if (job0) p1.gj = gamma_job(0);
    // the pass's predecessor is this call's prep kernel or the previous sweep's last kernel:
    // neither writes Z, so the first stages' Z loads may precede the PDL wait
    // (default only up to 2^26 elements: on c4a / c4b the prefetch changes nothing measurable and
    // the passes run the lean kernel instantiation instead, 5 us faster per c4a pass)
    double Pel = 1.0;
    for (int k = 0; k < N; ++k) Pel *= (double)s->dims[k];
    const bool zpre = path_flag("CP_STREAM_PREFETCH", Pel <= 67108864.0 ? 1 : 0) != 0;
    p1.prefetch = (zpre && p1.mma && p1.V >= 2) ? 1 : 0;
    if (!(skip & 128) && launch_stream(p1, cs) != cudaSuccess) return CP_ECUDA;
    ++launches;
    YLGeom yg;
    yg.R = R;
    yg.Gc = p1.Gc;
    yg.RB = p1.RB;
    yg.Wmax = p1.Wmax;
    yg.I0 = s->dims[0];
    yg.I1 = s->dims[1];
    yg.Q = p1.Q;
    yg.Qn = p1.Qn;
    yg.yl = w + L.yl;
    yg.edge = w + L.edge;
    double *mb = w + L.mbuf;
    if (!yl_inline) {
      if (launch_yl_fixup(yg, cs) != cudaSuccess) return CP_ECUDA;
      ++launches;
    }
    const bool ylsolve = path_flag("CP_YLSOLVE", 1) != 0;
    if (ylsolve) {
      // modes 0 and 1: M rows from Y_L, Gamma, Cholesky and the solves in one kernel each
      // (ylsolve.cu); Gamma^(0) from the Y_L pass's job when it ran, else factored in-block
      YLSolveArgs ya;
      memset(&ya, 0, sizeof(ya));
      ya.N = N;
      ya.R = R;
      ya.RSo = RS;
      ya.I0 = s->dims[0];
      ya.I1 = s->dims[1];
      ya.yl = w + L.yl;
      ya.pg = pg;
      ya.Ups = w + L.Ups;
      ya.status = w + L.status;
      for (int n = 0; n < 2; ++n) {
        ya.mode = n;
        ya.In = s->dims[n];
        ya.RS = RS;
        ya.Bfac = (n == 0) ? w + L.At[1] : A[0];
        ya.vec1 = (n == 1 && (s->dims[0] % 4) == 0 && aligned(A[0], 32)) ? 1 : 0;
        ya.gin = gp[0];
        ya.nin = grid_of[0];
        ya.linv = (n == 0 && job0) ? w + L.linv : nullptr;
        // mode 1 sums the Gram of A^(0)_new from mode 0's cluster partials (gin) and reads
        // Upsilon^(k >= 2) as totals (written by job 0 or by the mode-0 kernel)
        ya.total = nullptr;
        ya.ticket = reinterpret_cast<unsigned *>(w + L.status + kTicketSlot2);
        ya.ups_total = (n == 0) ? (steady ? (((1 << N) - 1) & ~1) : 0) : (((1 << N) - 1) & ~2);
        ya.F = (F != nullptr) ? F[n] : nullptr;
        ya.A = A[n];
        ya.At = w + L.At[n];
        ya.gcur = gp[n & 1];
        ya.dotF = w + L.dotF + (size_t)n * L.gp_max;
        grid_of[n] = ylsolve_clusters(s->dims[n]);
        if (launch_ylsolve(ya, cs) != cudaSuccess) return CP_ECUDA;
        launches += 1;
      }
    }
    // mode 0: M0 = sum_{i1} Y_L(:, i1, :) * A^(1)(i1, :)   (A^(2..) old: Gauss-Seidel order)
    if (!ylsolve) {
    if (!(skip & 2) && launch_ymm0(yg, A[1], w + L.m0part, cs) != cudaSuccess) return CP_ECUDA;
    ++launches;
    {
      // the mode-0 solve sums the ymm0 range partials (mode-0 partial layout, fixed order)
      ReduceGeom g0;
      memset(&g0, 0, sizeof(g0));
      g0.R = R;
      g0.Gc = ymm0_ranges(R, s->dims[1]);
      g0.RB = 1;
      g0.slots = 1;
      g0.mode0 = 1;
      g0.I1 = s->dims[0];
      g0.In_rows = s->dims[0];
      g0.part = w + L.m0part;
      int rpc0, sp0;
      ymm0_solve_blocking(R, s->dims[1], &rpc0, &sp0);
      if (!solve_mode(0, g0, rpc0, sp0, job0 ? w + L.linv : nullptr)) return CP_ECUDA;
    }
    // mode 1: M1 = sum_{i0} Y_L(i0, :, :) * A^(0)_new(i0, :); Gamma^(1) in an extra block
    GammaJob gj1;
    memset(&gj1, 0, sizeof(gj1));
    if (jobs) gj1 = gamma_job(1);
    if (!(skip & 64) && launch_ymm1(yg, A[0], mb, gj1, cs) != cudaSuccess) return CP_ECUDA;
    ++launches;
    if (!solve_mode(1, direct_geom(mb, s->dims[1], R), rpc_d, 1, jobs ? w + L.linv + (size_t)RR : nullptr))
      return CP_ECUDA;
    }  // !ylsolve
    // pass 2: modes >= 2 from Z x I0 x I1 contracted with the new A^(0), A^(1)
    StreamPlan p2 = L.p2_plan;
    p2.Z = Z;
    p2.At[0] = w + L.At[0];
    p2.At[1] = w + L.At[1];
    p2.At[2] = nullptr;
    p2.part = w + L.part;
    // Gamma^(2) rides in the pass's idle weight warp
    const bool job2 = jobs && p2.mma && p2.direct_w;
    if (job2) p2.gj = gamma_job(2);
    // N = 3: the mode-2 solve and the finalize run inside the pass (TailSolve, stream_mma.cuh
    // sweep_tail) -- no solve launch
    // sweep_tail) -- no solve launch.  CP_SWEEP_TAIL = 1 (default): only sweeps followed by another
    // steady sweep of the same call, with Upsilon^(2) and f left out (fin = 0: the next sweep's
    // Gamma^(0) job forms the Gram off the critical path; measured per steady sweep: c4a 421.5 ->
    // 419.0 us, c3 80.7 -> 75.9, c2 50.5 -> 46.9, c1 45.0 -> 41.0, tools/tail_ab.sh);
    // 2: every sweep (fin = 1 on a call's last sweep: measured 2-5 us slower than the solve launch it
    // replaces -- the last CTA's Gram and sums are a chain of L2 round trips -- so not the default).
    p2.prefetch = (zpre && p2.mma && p2.V >= 2) ? 1 : 0;  // (predecessor: the mode-1 solve)
    // (default only up to 2^26 elements: on c4a, 2^27, the ~4 us it saves per sweep are within the
    // run-to-run noise of the 420-us sweep, and the pass would carry the solve in its own time)
    const int tail_sel = path_flag("CP_SWEEP_TAIL", Pel <= 67108864.0 ? 1 : 0);
    const bool defer = defer_ok && deferred != nullptr && jobs && L.yl_plan.mma && L.yl_plan.direct_w;
    const bool tail = N == 3 && job2 && R <= 32 && p2.slots <= 32 && (tail_sel >= 2 || (tail_sel == 1 && defer)) &&
                      (int64_t)p2.nstages * p2.zst >= sweep_tail_doubles(R);
    if (tail) {
      TailSolve &t = p2.tail;
      t.on = 1;
      t.fin = defer ? 0 : 1;
      if (defer && deferred != nullptr) *deferred = true;
      t.dot_stride = L.gp_max;
      t.nsolve[0] = grid_of[0];
      t.nsolve[1] = grid_of[1];
      t.linv = w + L.linv + (size_t)2 * RR;
      t.F = (F != nullptr) ? F[2] : nullptr;
      t.A = A[2];
      t.At = w + L.At[2];
      t.rowdot = w + L.rowdot;
      t.dotF = w + L.dotF;
      t.Ups = w + L.Ups;
      t.normZ2 = normZ2;
      t.status = w + L.status;
      t.out = out;
      t.segtick = reinterpret_cast<unsigned *>(w + L.tailtick);
      t.gtick = t.segtick + L.maxI;
      t.gjflag = t.segtick + L.maxI + 1;
    }
    if (!(skip & 256) && launch_stream(p2, cs) != cudaSuccess) return CP_ECUDA;
    ++launches;
    if (tail) {
      // (solved and finalized by the pass)
    } else if (N == 3) {
      if (!solve_mode(2, reduce_geom(p2), L.rpc2, L.sp2, job2 ? w + L.linv + (size_t)2 * RR : nullptr))
        return CP_ECUDA;
    } else {
      if (launch_k(reduce_mttkrp_kernel, dim3(L.nyr), dim3(256), 0, cs, reduce_geom(p2), L.rpc2, L.sp2, w + L.yr) != cudaSuccess)
        return CP_ECUDA;
      ++launches;
      for (int m = 2; m < N; ++m) {
        YRArgs ya;
        memset(&ya, 0, sizeof(ya));
        ya.N = N;
        ya.R = R;
        ya.RS = RS;
        ya.mode = m;
        for (int k = 0; k < N; ++k) {
          ya.dims[k] = s->dims[k];
          ya.At[k] = w + L.At[k];
        }
        ya.YR = w + L.yr;
        ya.M = mb;
        // Gamma^(2) came with pass 2; Gamma^(m > 2) in an extra yr block when CP_GAMMA_JOBS=2
        // (measured: the yr kernels are too short to hide it)
        const bool jm = (m == 2) ? job2 : (jobs && knob("CP_GAMMA_JOBS", 1) >= 2);
        if (m > 2 && jm) ya.gj = gamma_job(m);
        if (launch_yr(ya, cs) != cudaSuccess) return CP_ECUDA;
        ++launches;
        if (!solve_mode(m, direct_geom(mb, s->dims[m], R), rpc_d, 1, jm ? w + L.linv + (size_t)m * RR : nullptr))
          return CP_ECUDA;
      }
    }
  } else {
    for (int n = 0; n < N; ++n) {
      StreamPlan p = L.plans[n];
      p.Z = Z;
      for (int k = 0; k < N; ++k) p.At[k] = w + L.At[k];
      p.part = w + L.part;
      if (launch_stream(p, cs) != cudaSuccess) return CP_ECUDA;
      ++launches;
      if (!solve_mode(n, reduce_geom(p), L.rpc[n], L.sp[n])) return CP_ECUDA;
    }
  }
  g_launches = launches;
  return CP_OK;
}

size_t cp_mode_product_workspace_bytes(int32_t N, const int64_t *dims, int32_t mode, int64_t J) {
  (void)N; (void)dims; (void)mode; (void)J;
  return 0;
}

int cp_mode_product(int32_t N, const int64_t *dims, const double *Z, int32_t mode, const double *U,
                    int64_t J, double *X, void *ws, size_t ws_bytes, cp_stream_t stream) {
  g_launches = 0;
  (void)ws; (void)ws_bytes;
  if (N < 1 || N > CP_MAX_N || dims == nullptr || mode < 0 || mode >= N || J < 1) return CP_EINVAL;
  if (!Z || !U || !X) return CP_EINVAL;
  double P = 1.0, PX = 1.0;
  for (int k = 0; k < N; ++k) {
    if (dims[k] < 1) return CP_EDIM;
    P *= (double)dims[k];
    PX *= (double)(k == mode ? J : dims[k]);
  }
  if (P >= 1125899906842624.0 || PX >= 1125899906842624.0) return CP_EDIM;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  const cudaError_t e = launch_mode_product(N, dims, Z, mode, U, J, X, cs);
  if (e != cudaSuccess) return e == cudaErrorInvalidConfiguration ? CP_EDIM : CP_ECUDA;
  g_launches = mode_product_launch_count(N, dims, mode);
  return CP_OK;
}

static bool use_small_sweep(const cp_shape &s);

// cp_fit (resid = true: f by the residual pass) and cp_gradient (resid = false: no residual
// pass, f by the expansion from the last mode's <M, A> and the Grams)
static int fit_impl(const cp_shape *s, const double *Z, const double *normZ2, const double *const *A,
                    const double *const *F, double *out, double *const *G, void *ws, size_t ws_bytes,
                    cp_stream_t stream, bool resid) {
  g_launches = 0;
  int st = check_shape(s, 2);
  if (st) return st;
  if (!Z || !normZ2 || !A || !out || !aligned(Z, 16)) return CP_EINVAL;
  for (int k = 0; k < s->N; ++k)
    if (A[k] == nullptr) return CP_EINVAL;
  const auto Lp = get_layout(*s);
  if (!Lp) return CP_EINVAL;
  const Layout &L = *Lp;
  if ((st = check_ws(L, ws, ws_bytes))) return st;
  double *w = static_cast<double *>(ws);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  const int N = s->N, R = s->R;
  if (!resid && use_small_sweep(*s)) {  // small tensor: the fused shared-memory kernel (gradient mode)
    if (launch_small_sweep(*s, Z, normZ2, const_cast<double *const *>(A), F, 1, out, cs, G, true) != cudaSuccess)
      return CP_ECUDA;
    g_launches = 1;
    return CP_OK;
  }
  PrepArgs pa;
  PrepGrams pg;
  fill_prep(*s, L, w, A, -1, true, nullptr, pa, pg);
  const bool yl_inline = L.tree && L.yl_plan.mma && knob("CP_YL_INLINE_FIX", 1);
  if (L.tree) {
    // u32 completion words zeroed by prep: the Y_L segment tickets (stream_mma.cuh
    // yl_complete_segment) and, contiguous after them, the tail solve's words (sweep_tail)
    const size_t z0 = yl_inline ? L.segtab : L.tailtick;
    pa.zero = reinterpret_cast<unsigned *>(w + z0);
    pa.nzero = (int)((L.tailtick - z0) * 2 + (size_t)L.maxI + 2);
  }
  // experiments only (-DCP_EXPERIMENTS builds): CP_SWEEP_SKIP bitmask drops launches (timing of
  // the rest; results wrong).  Always 0 in the shipped library.
  const int skip = knob("CP_SWEEP_SKIP", 0);
  if (!(skip & 1) && launch_prep(pa, cs) != cudaSuccess) return CP_ECUDA;
  int launches = 1;
  // residual pass 1/2 ||Z - [[A]]||^2 (eq:CPfunctional): one partial per CTA
  StreamPlan rp = L.resid;
  rp.Z = Z;
  for (int k = 0; k < N; ++k) rp.At[k] = w + L.At[k];
  rp.part = w + L.residp;
  if (resid) {
    if (launch_stream(rp, cs) != cudaSuccess) return CP_ECUDA;
    ++launches;
  }
  int ngrad[CP_MAX_N] = {0};
  // G^(n) = -M^(n) + A^(n) Gamma^(n) - F^(n) and its squared norm (eq:gradEqn, eq:gradConv)
  auto grad_mode = [&](int n, const ReduceGeom &rg, int rpc, int sp) -> bool {
    GradArgs ga;
    memset(&ga, 0, sizeof(ga));
    ga.N = N;
    ga.R = R;
    ga.mode = n;
    ga.rpc = rpc;
    ga.sp = sp;
    ga.In = s->dims[n];
    ga.rg = rg;
    ga.pg = pg;
    ga.A = A[n];
    ga.F = (F != nullptr) ? F[n] : nullptr;
    ga.Ups = w + L.Ups;
    ga.G = (G != nullptr) ? G[n] : nullptr;
    ga.gpart = w + L.gradp + (size_t)n * L.grad_max;
    ga.dpart = (!resid && n == N - 1) ? w + L.dotM : nullptr;  // (dotM holds gp_max >= ngrad)
    ngrad[n] = (int)ceil_div(s->dims[n], rpc);
    ++launches;
    return launch_k(gradient_kernel, dim3(ngrad[n]), dim3(256), 0, cs, ga) == cudaSuccess;
  };
  if (L.tree) {
    // all N MTTKRPs with the same factors through the dimension tree: 2 more passes over Z
    // (the Y_L pass and the mode-2 pass of Z viewed as I0 x I1 x J), as in cp_als_sweep
    const int rpc_d = 256 / R > 0 ? 256 / R : 1;
    StreamPlan p1 = L.yl_plan;
    p1.Z = Z;
    for (int k = 0; k < N; ++k) p1.At[k] = w + L.At[k];
    p1.yl = w + L.yl;
    p1.edge = w + L.edge;
    p1.segcnt = yl_inline ? reinterpret_cast<unsigned *>(w + L.segtab) : nullptr;
    p1.part = nullptr;
    if (!(skip & 128) && launch_stream(p1, cs) != cudaSuccess) return CP_ECUDA;
    ++launches;
    YLGeom yg;
    yg.R = R;
    yg.Gc = p1.Gc;
    yg.RB = p1.RB;
    yg.Wmax = p1.Wmax;
    yg.I0 = s->dims[0];
    yg.I1 = s->dims[1];
    yg.Q = p1.Q;
    yg.Qn = p1.Qn;
    yg.yl = w + L.yl;
    yg.edge = w + L.edge;
    double *mb = w + L.mbuf;
    if (!yl_inline) {
      if (launch_yl_fixup(yg, cs) != cudaSuccess) return CP_ECUDA;
      ++launches;
    }
    if (!(skip & 2) && launch_ymm0(yg, A[1], w + L.m0part, cs) != cudaSuccess) return CP_ECUDA;
    ++launches;
    {
      ReduceGeom g0;
      memset(&g0, 0, sizeof(g0));
      g0.R = R;
      g0.Gc = ymm0_ranges(R, s->dims[1]);
      g0.RB = 1;
      g0.slots = 1;
      g0.mode0 = 1;
      g0.I1 = s->dims[0];
      g0.In_rows = s->dims[0];
      g0.part = w + L.m0part;
      int rpc0, sp0;
      ymm0_solve_blocking(R, s->dims[1], &rpc0, &sp0);
      if (!grad_mode(0, g0, rpc0, sp0)) return CP_ECUDA;
    }
    GammaJob nojob;
    memset(&nojob, 0, sizeof(nojob));
    if (launch_ymm1(yg, A[0], mb, nojob, cs) != cudaSuccess) return CP_ECUDA;
    ++launches;
    if (!grad_mode(1, direct_geom(mb, s->dims[1], R), rpc_d, 1)) return CP_ECUDA;
    StreamPlan p2 = L.p2_plan;
    p2.Z = Z;
    p2.At[0] = w + L.At[0];
    p2.At[1] = w + L.At[1];
    p2.At[2] = nullptr;
    p2.part = w + L.part;
    if (launch_stream(p2, cs) != cudaSuccess) return CP_ECUDA;
    ++launches;
    if (N == 3) {
      if (!grad_mode(2, reduce_geom(p2), L.rpc2, L.sp2)) return CP_ECUDA;
    } else {
      if (launch_k(reduce_mttkrp_kernel, dim3(L.nyr), dim3(256), 0, cs, reduce_geom(p2), L.rpc2, L.sp2,
                   w + L.yr) != cudaSuccess)
        return CP_ECUDA;
      ++launches;
      for (int m = 2; m < N; ++m) {
        YRArgs ya;
        memset(&ya, 0, sizeof(ya));
        ya.N = N;
        ya.R = R;
        ya.RS = R + (R & 1);
        ya.mode = m;
        for (int k = 0; k < N; ++k) {
          ya.dims[k] = s->dims[k];
          ya.At[k] = w + L.At[k];
        }
        ya.YR = w + L.yr;
        ya.M = mb;
        if (launch_yr(ya, cs) != cudaSuccess) return CP_ECUDA;
        ++launches;
        if (!grad_mode(m, direct_geom(mb, s->dims[m], R), rpc_d, 1)) return CP_ECUDA;
      }
    }
  } else {
    for (int n = 0; n < N; ++n) {
      StreamPlan p = L.plans[n];
      p.Z = Z;
      for (int k = 0; k < N; ++k) p.At[k] = w + L.At[k];
      p.part = w + L.part;
      if (launch_stream(p, cs) != cudaSuccess) return CP_ECUDA;
      ++launches;
      if (!grad_mode(n, reduce_geom(p), L.rpc[n], L.sp[n])) return CP_ECUDA;
    }
  }
  FitFinalArgs fa;
  memset(&fa, 0, sizeof(fa));
  fa.N = N;
  fa.nresid = rp.Gc * rp.RB;
  fa.gstride = L.grad_max;
  for (int n = 0; n < N; ++n) fa.ngrad[n] = ngrad[n];
  fa.resid = rp.part;
  fa.gpart = w + L.gradp;
  fa.normZ2 = normZ2;
  fa.out = out;
  if (!resid) {
    fa.nresid = 0;
    fa.expand = 1;
    fa.R = R;
    fa.ndot = ngrad[N - 1];
    fa.dpart = w + L.dotM;
    fa.pg = pg;
  }
  if (launch_k(finalize_fit_kernel, dim3(1), dim3(256), 0, cs, fa) != cudaSuccess) return CP_ECUDA;
  g_launches = launches + 1;
  return CP_OK;
}

int cp_fit(const cp_shape *s, const double *Z, const double *normZ2, const double *const *A,
           const double *const *F, double *out, double *const *G, void *ws, size_t ws_bytes,
           cp_stream_t stream) {
  return fit_impl(s, Z, normZ2, A, F, out, G, ws, ws_bytes, stream, true);
}

int cp_gradient(const cp_shape *s, const double *Z, const double *normZ2, const double *const *A,
                const double *const *F, double *out, double *const *G, void *ws, size_t ws_bytes,
                cp_stream_t stream) {
  return fit_impl(s, Z, normZ2, A, F, out, G, ws, ws_bytes, stream, false);
}

int cp_als_sweeps_then_gradient(const cp_shape *s, const double *Z, const double *normZ2,
                                double *const *A, const double *const *F, int32_t nsweeps,
                                int32_t flags, double *out, const double *const *gF, double *gout,
                                double *const *G, void *ws, size_t ws_bytes, cp_stream_t stream) {
  g_launches = 0;
  if (!gout) return CP_EINVAL;
  int st = check_shape(s, 2);
  if (st) return st;
  // small tensors beyond the tiny kernel's shapes: sweeps and the gradient pass in one launch of
  // the fused kernel
  if (Z && normZ2 && A && out && aligned(Z, 16) && nsweeps >= 1 && !(flags & ~CP_SWEEPS_NORMALIZE) &&
      use_small_sweep(*s) && !(path_flag("CP_TINY_SWEEP", 1) != 0 && tiny_sweep_ok(*s)) &&
      path_flag("CP_SWEEPS_GRAD_FUSED", 1) != 0) {
    for (int k = 0; k < s->N; ++k)
      if (A[k] == nullptr) return CP_EINVAL;
    const auto Lp = get_layout(*s);
    if (!Lp) return CP_EINVAL;
    if ((st = check_ws(*Lp, ws, ws_bytes))) return st;
    if (launch_small_sweep(*s, Z, normZ2, A, F, nsweeps, out, reinterpret_cast<cudaStream_t>(stream), G, false,
                           (flags & CP_SWEEPS_NORMALIZE) != 0, gout, gF) != cudaSuccess)
      return CP_ECUDA;
    g_launches = 1;
    return CP_OK;
  }
  if ((st = cp_als_sweeps(s, Z, normZ2, A, F, nsweeps, flags, out, ws, ws_bytes, stream))) return st;
  const int n1 = g_launches;
  if ((st = cp_gradient(s, Z, normZ2, A, gF, gout, G, ws, ws_bytes, stream))) return st;
  g_launches += n1;
  return CP_OK;
}

int cp_normalize_sort(const cp_shape *s, double *const *A, int32_t sort, double *lambda, void *ws,
                      size_t ws_bytes, cp_stream_t stream) {
  g_launches = 0;
  int st = check_shape(s, 1);
  if (st) return st;
  if (!A || !ws || !aligned(ws, 256)) return CP_EINVAL;
  NormArgs a;
  memset(&a, 0, sizeof(a));
  a.N = s->N;
  a.R = s->R;
  a.sort = sort ? 1 : 0;
  int64_t off = 0;
  for (int n = 0; n < s->N; ++n) {
    if (!A[n]) return CP_EINVAL;
    a.dims[n] = s->dims[n];
    a.A[n] = A[n];
    a.off[n] = off;
    off += s->dims[n] * s->R;
  }
  if ((size_t)off * sizeof(double) > ws_bytes) return CP_EWORKSPACE;
  a.tmp = static_cast<double *>(ws);
  a.lambda = lambda;
  if (launch_normalize_sort(a, reinterpret_cast<cudaStream_t>(stream)) != cudaSuccess) return CP_ECUDA;
  g_launches = 1;
  return CP_OK;
}

int cp_last_launch_count(void) { return g_launches; }

int cp_profile_enable(int enable) {
  if (enable && !g_prof_init) {
    for (int i = 0; i < 2 * kProfMax; ++i)
      if (cudaEventCreate(&g_prof_ev[i]) != cudaSuccess) return CP_ECUDA;
    g_prof_init = true;
  }
  g_prof_on = enable != 0;
  g_prof_n = 0;
  return CP_OK;
}

int cp_profile_read(int64_t *launches, double *total_ms, double *alg_bytes) {
  if (!launches || !total_ms || !alg_bytes) return CP_EINVAL;
  double ms = 0.0, bytes = 0.0;
  for (int i = 0; i < g_prof_n; ++i) {
    float t = 0.f;
    if (cudaEventSynchronize(g_prof_ev[2 * i + 1]) != cudaSuccess) return CP_ECUDA;
    if (cudaEventElapsedTime(&t, g_prof_ev[2 * i], g_prof_ev[2 * i + 1]) != cudaSuccess) return CP_ECUDA;
    ms += t;
    bytes += g_prof_bytes[i];
  }
  *launches = g_prof_n;
  *total_ms = ms;
  *alg_bytes = bytes;
  g_prof_n = 0;
  return CP_OK;
}

const char *cp_status_string(int code) {
  switch (code) {
    case CP_OK: return "ok";
    case CP_EINVAL: return "invalid argument";
    case CP_EDIM: return "invalid dimension";
    case CP_ENOTSPD: return "Gamma not positive definite (Cholesky pivot <= 0)";
    case CP_ECUDA: return "CUDA launch failure";
    case CP_EWORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

int cp_version(void) { return CP_VERSION; }

}  // extern "C"
