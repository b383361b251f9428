// mg_driver.cu -- the multigrid CP driver of De Sterck & Miller (arXiv 1111.6091) as host C++
// on top of the C ABI of this library.
//
//   setup phase  : CP-AMG-mult V-cycles (Algorithm 1): ALS relaxation on test
//                  blocks and boot factors, geometric coarsening, weighted LS
//                  interpolation (eq:LSQinterp, eq:interpweights P:236-247), B = P^T P = L L^T,
//                  Phat = P L^{-T}, R = Phat^T, Galerkin tensor Z x_n R
//                  (eq:ctensor_transformed), coarse-grid correction Phat A_c (eq:CGC_new).
//   FMG          : FMG-CP-FAS (Algorithm 3).
//   solve phase  : CP-FAS V-cycles (Algorithm 2): BNGS with RHS (eq:relaxinnersolve),
//                  F_c = H_c(A~_c) + R(F - H(A)) (eq:FASrhs), A += Phat (A_c - A~_c) (eq:FASCGC);
//                  normalization + ordering on the finest level only.
//   combination  : <= 5 setup cycles, stagnation test after 3 (eq:stagnation), optional FMG with
//                  a down-sweep rebuild, solve cycles until g < tau with the one-time rebuild on
//                  solve stagnation.
// Every tensor-sized operation is a call into the kernels of this library; the host only builds
// the transfer operators (O(I * I_c) per mode) and reads g once per cycle.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "../../include/cp.h"
#include "cp_internal.cuh"
#include "mg_kernels.cuh"

namespace cpk {
namespace {

constexpr int kMaxTest = 8;
constexpr int kMaxLevels = 40;
// device `out` words of the relaxation calls (4 doubles each): every cp_als_sweep(s) call of a
// cycle writes its own slot, and the host checks every slot's status at the next stopping test
// (which synchronizes anyway), so a Cholesky failure on any level is reported (CP_ENOTSPD)
constexpr int kOutSlots = 4096;

// CP_MG_STRUCTURED=0 (path selector): Galerkin tensors by the dense mode product
static bool structured_restriction() { return path_flag("CP_MG_STRUCTURED", 1) != 0; }

struct Arena {
  char *base = nullptr;
  size_t cap = 0, off = 0;
  bool dry = true;
  double *take(size_t n) {
    off = (off + 255) & ~(size_t)255;
    double *p = dry ? nullptr : reinterpret_cast<double *>(base + off);
    off += n * sizeof(double);
    return p;
  }
};

struct Level {
  cp_shape s;
  int64_t P = 0;
  bool has_next = false;
  bool coarsen[CP_MAX_N] = {};
  int64_t Ic[CP_MAX_N] = {};  // next-level sizes
  const double *Z = nullptr;
  double *zbuf = nullptr;
  double *nz2 = nullptr;
  double *A[CP_MAX_N] = {}, *F[CP_MAX_N] = {}, *H[CP_MAX_N] = {}, *Atil[CP_MAX_N] = {},
         *tmp[CP_MAX_N] = {}, *prev[CP_MAX_N] = {};
  double *T[kMaxTest][CP_MAX_N] = {};
  double *Ph[CP_MAX_N] = {}, *Rt[CP_MAX_N] = {};
  double *wl[CP_MAX_N] = {}, *wr[CP_MAX_N] = {};  // F-row weights of P (cp_restrict_structured)
};

struct MG {
  cp_mg_params prm;
  int N = 0, R = 0, nt = 0, L = 0;
  Level lv[kMaxLevels];
  double *scratch[2] = {nullptr, nullptr};
  double *out_fit = nullptr, *out_slots = nullptr;
  int nslot = 0, slot_hi = 0;  // next slot; slots used so far (checked at every stopping test)
  std::vector<double> h_slots;
  int failed_mode = -1;
  void *ws = nullptr;
  size_t ws_bytes = 0;
  cudaStream_t st = nullptr;
  cp_stream_t cst = nullptr;
  int err = CP_OK;
  double fit_seconds = 0.0;
  std::vector<double> h_fit;
  cudaEvent_t fev[2] = {nullptr, nullptr};  // device time of the stopping-test cp_gradient calls
  void destroy_events() {
    for (cudaEvent_t &e : fev)
      if (e) {
        cudaEventDestroy(e);
        e = nullptr;
      }
  }

  // ------------------------------------------------------------ planning / allocation
  bool plan(const cp_shape &s0, const cp_mg_params &p) {
    prm = p;
    N = s0.N;
    R = s0.R;
    nt = p.n_test;
    if (nt < 1 || nt > kMaxTest) return false;
    const int64_t coarsest = p.coarsest > 0 ? p.coarsest : 2 * (int64_t)R;
    lv[0].s = s0;
    L = 1;
    for (;;) {
      Level &c = lv[L - 1];
      c.P = 1;
      for (int n = 0; n < N; ++n) c.P *= c.s.dims[n];
      bool any = false;
      for (int n = 0; n < N; ++n) {
        c.coarsen[n] = c.s.dims[n] > coarsest;
        c.Ic[n] = c.coarsen[n] ? (c.s.dims[n] + 1) / 2 : c.s.dims[n];
        any = any || c.coarsen[n];
      }
      c.has_next = any;
      if (!any) break;
      if (L >= kMaxLevels) return false;
      Level &nx = lv[L];
      nx.s = c.s;
      for (int n = 0; n < N; ++n) nx.s.dims[n] = c.Ic[n];
      ++L;
    }
    return true;
  }

  size_t layout(Arena &a) {
    size_t wsb = 0;
    for (int l = 0; l < L; ++l) {
      Level &v = lv[l];
      if (l > 0) v.zbuf = a.take(v.P);
      v.nz2 = a.take(1);
      for (int n = 0; n < N; ++n) {
        const size_t m = (size_t)v.s.dims[n] * R;
        v.A[n] = (l == 0) ? nullptr : a.take(m);  // level 0 uses the caller's A
        v.F[n] = a.take(m);
        v.H[n] = a.take(m);
        v.Atil[n] = a.take(m);
        v.tmp[n] = a.take(m);
        v.prev[n] = a.take(m);
        for (int t = 0; t < nt; ++t) v.T[t][n] = a.take(m);
        if (v.has_next && v.coarsen[n]) {
          v.Ph[n] = a.take((size_t)v.s.dims[n] * v.Ic[n]);
          v.Rt[n] = a.take((size_t)v.s.dims[n] * v.Ic[n]);
          v.wl[n] = a.take((size_t)v.s.dims[n]);
          v.wr[n] = a.take((size_t)v.s.dims[n]);
          const size_t rw = cp_restrict_workspace_bytes(N, v.s.dims, n);
          if (rw > wsb) wsb = rw;
        }
      }
      const size_t w = cp_workspace_bytes(&v.s);
      if (w == 0) return 0;
      if (w > wsb) wsb = w;
    }
    scratch[0] = a.take((size_t)(lv[0].P / 2 + 1));
    scratch[1] = a.take((size_t)(lv[0].P / 4 + 1));
    out_fit = a.take(2 + N);
    out_slots = a.take((size_t)4 * kOutSlots);
    a.off = (a.off + 255) & ~(size_t)255;
    ws = a.dry ? nullptr : a.base + a.off;
    ws_bytes = wsb;
    a.off += wsb;
    return a.off;
  }

  bool ok(int rc) {
    if (rc != CP_OK && err == CP_OK) err = rc;
    return err == CP_OK;
  }
  // the out word of the next relaxation call (wraps: slots are re-read at every stopping test,
  // and a cycle issues far fewer than kOutSlots relaxation calls)
  double *next_out() {
    double *o = out_slots + 4 * (size_t)(nslot % kOutSlots);
    ++nslot;
    if (nslot > slot_hi) slot_hi = nslot < kOutSlots ? nslot : kOutSlots;
    return o;
  }
  // after fit()'s read-back: CP_ENOTSPD if any relaxation since the solve began failed
  void check_slots() {
    if (err != CP_OK) return;
    for (int k = 0; k < (int)h_slots.size() / 4; ++k)
      if (h_slots[4 * k + 2] != 0.0) {
        err = CP_ENOTSPD;
        failed_mode = (int)h_slots[4 * k + 3];
        return;
      }
  }
  void copy(double *dst, const double *src, size_t n) {
    if (err == CP_OK && cudaMemcpyAsync(dst, src, n * 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      err = CP_ECUDA;
  }
  void lincomb(double *out, double a, const double *x, double b, const double *y, int64_t n) {
    if (err == CP_OK && launch_lincomb(out, a, x, b, y, n, st) != cudaSuccess) err = CP_ECUDA;
  }

  // ------------------------------------------------------------ building blocks
  // ALS relaxation of the setup phase: sweep + normalization, every level
  void relax_setup(int l, double *const *A, int sweeps) {
    Level &v = lv[l];
    // sweep + normalization (no sort) nu times: one fused launch on small levels
    if (sweeps > 0)
      ok(cp_als_sweeps(&v.s, v.Z, v.nz2, A, nullptr, sweeps, CP_SWEEPS_NORMALIZE, next_out(), ws, ws_bytes, cst));
  }
  // BNGS with RHS (eq:relaxinnersolve); finest level: normalize + sort
  void relax_fas(int l, double *const *A, const double *const *F, int sweeps) {
    Level &v = lv[l];
    if (l > 0) {  // coarse levels: no normalization between sweeps -> one call (fused when small)
      if (sweeps > 0) ok(cp_als_sweeps(&v.s, v.Z, v.nz2, A, F, sweeps, 0, next_out(), ws, ws_bytes, cst));
      return;
    }
    for (int k = 0; k < sweeps && err == CP_OK; ++k) {
      ok(cp_als_sweep(&v.s, v.Z, v.nz2, A, F, next_out(), ws, ws_bytes, cst));
      ok(cp_normalize_sort(&v.s, A, 1, nullptr, ws, ws_bytes, cst));
    }
  }
  // g (eq:gradConv) at level l; optional G^(n) = H^(n)(A) into G (F = 0)
  // (host synchronizing: the value is read on the host).  fit_seconds accumulates the DEVICE time
  // of the cp_gradient call (CUDA events around it), not the host wait for earlier queued work.
  double fit(int l, double *const *A, double *const *G, double *gradnorm2 = nullptr) {
    Level &v = lv[l];
    if (err != CP_OK) return NAN;
    if (!fev[0] && (cudaEventCreate(&fev[0]) != cudaSuccess || cudaEventCreate(&fev[1]) != cudaSuccess)) {
      err = CP_ECUDA;
      return NAN;
    }
    cudaEventRecord(fev[0], st);
    ok(cp_gradient(&v.s, v.Z, v.nz2, A, nullptr, out_fit, G, ws, ws_bytes, cst));  // NEXT-2: no residual pass
    cudaEventRecord(fev[1], st);
    h_fit.assign(2 + N, NAN);
    h_slots.assign((size_t)4 * slot_hi, 0.0);
    if (err == CP_OK &&
        (cudaMemcpyAsync(h_fit.data(), out_fit, (2 + N) * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
         (slot_hi > 0 &&
          cudaMemcpyAsync(h_slots.data(), out_slots, h_slots.size() * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess)))
      err = CP_ECUDA;
    if (err == CP_OK && cudaStreamSynchronize(st) != cudaSuccess) err = CP_ECUDA;
    float ms = 0.f;
    if (err == CP_OK && cudaEventElapsedTime(&ms, fev[0], fev[1]) == cudaSuccess) fit_seconds += 1e-3 * ms;
    check_slots();
    if (err != CP_OK) return NAN;
    if (gradnorm2)
      for (int n = 0; n < N; ++n) gradnorm2[n] = h_fit[2 + n];
    return h_fit[1];
  }
  // G^(n) = H^(n)(A) at level l, enqueued only (no host synchronization; graph-capturable)
  void grad(int l, double *const *A, double *const *G) {
    Level &v = lv[l];
    if (err != CP_OK) return;
    ok(cp_gradient(&v.s, v.Z, v.nz2, A, nullptr, out_fit, G, ws, ws_bytes, cst));
  }
  // The factor-sized transfers of level l, every mode in ONE launch (xfer_kernel): restriction
  // R^(n) = Phat^(n)T (Ic x I) or interpolation Phat^(n) (I x Ic) of the coarsened modes, identity
  // otherwise (eq:coarseapprox_new, eq:CGC_new, eq:FASrhs, eq:FASCGC)
  XferArgs xfer_args(int l, int op, bool down) {
    Level &v = lv[l];
    XferArgs a;
    memset(&a, 0, sizeof(a));
    a.N = N;
    a.R = R;
    a.op = op;
    for (int n = 0; n < N; ++n) {
      a.coarsen[n] = v.coarsen[n] ? 1 : 0;
      a.rows_in[n] = down ? v.s.dims[n] : v.Ic[n];
      a.rows_out[n] = down ? v.Ic[n] : v.s.dims[n];
      a.T[n] = v.coarsen[n] ? (down ? v.Rt[n] : v.Ph[n]) : nullptr;
    }
    return a;
  }
  void xfer(XferArgs &a) {
    if (err == CP_OK && launch_xfer(a, st) != cudaSuccess) err = CP_ECUDA;
  }
  // dst (level l+1 sizes) = R^(n) src^(n) for coarsened modes, copy otherwise
  void restrict_(int l, double *const *src, double *const *dst) {
    XferArgs a = xfer_args(l, kXferApply, true);
    for (int n = 0; n < N; ++n) {
      a.x[n] = src[n];
      a.dst[n] = dst[n];
    }
    xfer(a);
  }
  // dst (level l sizes) = Phat^(n) src^(n) for coarsened modes, copy otherwise
  void interp(int l, double *const *src, double *const *dst) {
    XferArgs a = xfer_args(l, kXferApply, false);
    for (int n = 0; n < N; ++n) {
      a.x[n] = src[n];
      a.dst[n] = dst[n];
    }
    xfer(a);
  }

  // Transfer operators of level l fitted to the test blocks (and the boot factors
  // unless first), then the Galerkin tensor of level l+1.
  void build_ops(int l, bool first) {
    Level &v = lv[l];
    // LS weights: w = ||A^(n)||^2 / ||G^(n)||^2 per factor matrix (eq:interpweights)
    std::vector<std::vector<double>> gn(nt + 1, std::vector<double>(N, 0.0));
    for (int t = 0; t < nt; ++t) fit(l, v.T[t], nullptr, gn[t].data());
    if (!first) fit(l, v.A, nullptr, gn[nt].data());
    if (err != CP_OK) return;
    for (int n = 0; n < N; ++n) {
      if (!v.coarsen[n]) continue;
      const int64_t I = v.s.dims[n], Ic = v.Ic[n];
      const int nf = first ? nt : nt + 1;
      // host copies of the fitted factor matrices (I x R col-major each)
      std::vector<double> U((size_t)nf * I * R);
      for (int t = 0; t < nf; ++t) {
        const double *src = (t < nt) ? v.T[t][n] : v.A[n];
        if (cudaMemcpyAsync(U.data() + (size_t)t * I * R, src, (size_t)I * R * 8, cudaMemcpyDeviceToHost,
                            st) != cudaSuccess)
          err = CP_ECUDA;
      }
      if (err != CP_OK || cudaStreamSynchronize(st) != cudaSuccess) {
        err = CP_ECUDA;
        return;
      }
      std::vector<double> wt(nf);
      for (int t = 0; t < nf; ++t) {
        double a2 = 0.0;
        for (int64_t e = 0; e < I * R; ++e) a2 += U[(size_t)t * I * R + e] * U[(size_t)t * I * R + e];
        wt[t] = a2 / gn[t][n];
      }
      // P: C points 2c (0-based) -> coarse c; F point f interpolates from (f-1)/2 and (f+1)/2
      // (one-sided at an even right end, reading R17); weights by weighted LS over
      // the nf*R fitted vectors, normal equations
      std::vector<int64_t> c0(I), c1(I);
      std::vector<double> w0(I), w1(I);
      for (int64_t i = 0; i < I; ++i) {
        if ((i & 1) == 0) {
          c0[i] = i / 2;
          c1[i] = -1;
          w0[i] = 1.0;
          w1[i] = 0.0;
          continue;
        }
        c0[i] = (i - 1) / 2;
        c1[i] = (i + 1 < I) ? (i + 1) / 2 : -1;
        double a00 = 0, a01 = 0, a11 = 0, b0 = 0, b1 = 0;
        for (int t = 0; t < nf; ++t)
          for (int r = 0; r < R; ++r) {
            const double *u = U.data() + (size_t)t * I * R + (size_t)r * I;
            const double x0 = u[i - 1], y = u[i];
            const double x1 = (c1[i] >= 0) ? u[i + 1] : 0.0;
            a00 += wt[t] * x0 * x0;
            a01 += wt[t] * x0 * x1;
            a11 += wt[t] * x1 * x1;
            b0 += wt[t] * x0 * y;
            b1 += wt[t] * x1 * y;
          }
        if (c1[i] >= 0) {
          const double det = a00 * a11 - a01 * a01;
          w0[i] = (a11 * b0 - a01 * b1) / det;
          w1[i] = (a00 * b1 - a01 * b0) / det;
        } else {
          w0[i] = b0 / a00;
          w1[i] = 0.0;
        }
      }
      // B = P^T P (tridiagonal: diagonal d, sub-diagonal e), B = L L^T with L bidiagonal
      std::vector<double> d(Ic, 0.0), e(Ic, 0.0), ld(Ic), le(Ic);
      for (int64_t i = 0; i < I; ++i) {
        d[c0[i]] += w0[i] * w0[i];
        if (c1[i] >= 0) {
          d[c1[i]] += w1[i] * w1[i];
          e[c1[i]] += w0[i] * w1[i];  // B(c1, c1-1) with c0 = c1 - 1
        }
      }
      for (int64_t j = 0; j < Ic; ++j) {
        le[j] = (j > 0) ? e[j] / ld[j - 1] : 0.0;
        const double piv = d[j] - le[j] * le[j];
        if (!(piv > 0.0)) {
          err = CP_ENOTSPD;
          return;
        }
        ld[j] = std::sqrt(piv);
      }
      // Phat = P L^{-T}: row i of Phat solves L y = p_i (p_i has <= 2 nonzeros)
      std::vector<double> Ph((size_t)I * Ic, 0.0), Rt((size_t)I * Ic, 0.0);
      for (int64_t i = 0; i < I; ++i) {
        double yprev = 0.0;
        for (int64_t j = c0[i]; j < Ic; ++j) {
          double pij = (j == c0[i]) ? w0[i] : ((j == c1[i]) ? w1[i] : 0.0);
          const double y = (pij - ((j > c0[i]) ? le[j] * yprev : 0.0)) / ld[j];
          Ph[(size_t)i + (size_t)I * j] = y;
          Rt[(size_t)j + (size_t)Ic * i] = y;
          yprev = y;
        }
      }
      if (cudaMemcpyAsync(v.Ph[n], Ph.data(), Ph.size() * 8, cudaMemcpyHostToDevice, st) != cudaSuccess ||
          cudaMemcpyAsync(v.Rt[n], Rt.data(), Rt.size() * 8, cudaMemcpyHostToDevice, st) != cudaSuccess ||
          cudaMemcpyAsync(v.wl[n], w0.data(), (size_t)I * 8, cudaMemcpyHostToDevice, st) != cudaSuccess ||
          cudaMemcpyAsync(v.wr[n], w1.data(), (size_t)I * 8, cudaMemcpyHostToDevice, st) != cudaSuccess ||
          cudaStreamSynchronize(st) != cudaSuccess) {
        err = CP_ECUDA;
        return;
      }
    }
    // Galerkin tensor Z_{l+1} = Z_l x_{n in I_c} R^(n), modes in increasing order
    Level &nx = lv[l + 1];
    const double *src = v.Z;
    int64_t cur[CP_MAX_N];
    for (int n = 0; n < N; ++n) cur[n] = v.s.dims[n];
    int remaining = 0;
    for (int n = 0; n < N; ++n) remaining += v.coarsen[n] ? 1 : 0;
    int ping = 0;
    for (int n = 0; n < N && err == CP_OK; ++n) {
      if (!v.coarsen[n]) continue;
      --remaining;
      double *dst = (remaining == 0) ? nx.zbuf : scratch[ping];
      // Galerkin tensor by the structured operator (3-tap gather + bidiagonal
      // substitution, HBM-bound); CP_MG_STRUCTURED=0: the dense product with Phat^T
      if (structured_restriction())
        ok(cp_restrict_structured(N, cur, src, n, v.wl[n], v.wr[n], dst, ws, ws_bytes, cst));
      else
        ok(cp_mode_product(N, cur, src, n, v.Rt[n], v.Ic[n], dst, nullptr, 0, cst));
      cur[n] = v.Ic[n];
      src = dst;
      ping ^= 1;
    }
    nx.Z = nx.zbuf;
    cp_shape s1 = nx.s;
    s1.R = 1;
    ok(cp_norm2(&s1, nx.Z, nx.nz2, ws, ws_bytes, cst));
  }

  // Algorithm 1 (CP-AMG-mult).  update_boot = false: the down-sweep rebuild of P:490-492
  // (test blocks relaxed, boot factors fitted but not updated, no up-sweep).
  void setup_cycle(int l, bool first, bool update_boot) {
    Level &v = lv[l];
    if (err != CP_OK) return;
    if (!v.has_next) {
      if (update_boot) relax_setup(l, v.A, prm.nuc_setup);
      return;
    }
    for (int t = 0; t < nt; ++t) relax_setup(l, v.T[t], prm.nu1_setup);
    if (update_boot) relax_setup(l, v.A, prm.nu1_setup);
    build_ops(l, first);
    Level &nx = lv[l + 1];
    restrict_(l, v.A, nx.A);
    for (int t = 0; t < nt; ++t) restrict_(l, v.T[t], nx.T[t]);
    setup_cycle(l + 1, first, update_boot);
    if (update_boot && err == CP_OK) {
      interp(l, nx.A, v.A);
      relax_setup(l, v.A, prm.nu2_setup);
    }
  }

  // Algorithm 2 (CP-FAS); F == nullptr means F = 0
  void fas_cycle(int l, double *const *F) {
    Level &v = lv[l];
    if (err != CP_OK) return;
    if (!v.has_next) {
      relax_fas(l, v.A, F, prm.nuc_solve);
      return;
    }
    Level &nx = lv[l + 1];
    if (l > 0 && prm.nu1_solve > 0) {
      // pre-relaxation and H(A) at the relaxed iterate as one call (one launch on small levels;
      // bitwise the two calls)
      ok(cp_als_sweeps_then_gradient(&v.s, v.Z, v.nz2, v.A, F, prm.nu1_solve, 0, next_out(), nullptr, out_fit, v.H,
                                     ws, ws_bytes, cst));
      restrict_(l, v.A, nx.Atil);   // A~_c
    } else {
      relax_fas(l, v.A, F, prm.nu1_solve);
      restrict_(l, v.A, nx.Atil);   // A~_c
      grad(l, v.A, v.H);            // H(A)
    }
    grad(l + 1, nx.Atil, nx.H);     // H_c(A~_c)
    {                               // F_c = H_c(A~_c) + R (F - H(A))  (eq:FASrhs);  A_c = A~_c
      XferArgs a = xfer_args(l, kXferFasRhs, true);
      for (int n = 0; n < N; ++n) {
        a.x[n] = v.H[n];
        a.y[n] = F ? F[n] : nullptr;
        a.z[n] = nx.H[n];
        a.w[n] = nx.Atil[n];
        a.dst[n] = nx.F[n];
        a.dst2[n] = nx.A[n];
      }
      xfer(a);
    }
    fas_cycle(l + 1, nx.F);
    {                               // A += Phat (A_c - A~_c)  (eq:FASCGC)
      XferArgs a = xfer_args(l, kXferCorrect, false);
      for (int n = 0; n < N; ++n) {
        a.x[n] = nx.A[n];
        a.y[n] = nx.Atil[n];
        a.dst[n] = v.A[n];
      }
      xfer(a);
    }
    relax_fas(l, v.A, F, prm.nu2_solve);
  }

  // Algorithm 3 (FMG-CP-FAS)
  void fmg(const double *const *Afmg) {
    Level &c = lv[L - 1];
    for (int n = 0; n < N; ++n) copy(c.A[n], Afmg[n], (size_t)c.s.dims[n] * R);
    relax_setup(L - 1, c.A, prm.nu_fmg);
    for (int l = L - 1; l >= 1 && err == CP_OK; --l) {
      interp(l - 1, lv[l].A, lv[l - 1].A);
      fas_cycle(l - 1, nullptr);
    }
  }
};

}  // namespace
}  // namespace cpk

using namespace cpk;

extern "C" {

void cp_mg_default_params(cp_mg_params *p) {
  if (!p) return;
  p->nu1_setup = 5;
  p->nu2_setup = 5;
  p->nuc_setup = 100;
  p->n_test = 2;
  p->nu1_solve = 1;
  p->nu2_solve = 1;
  p->nuc_solve = 50;
  p->max_setup_cycles = 5;
  p->min_setup_cycles = 3;
  p->stagnation_eps = 0.1;
  p->use_fmg = 0;
  p->nu_fmg = 50;
  p->max_cycles = 500;
  p->tol = 1e-10;
  p->coarsest = 0;
  p->solve_stagnation_after = 5;
  p->max_trace = 0;
  p->fmg_guard = 0;
}

size_t cp_mg_workspace_bytes(const cp_shape *s, const cp_mg_params *p) {
  if (!s || !p || s->N < 2 || s->N > CP_MAX_N || s->R < 1 || s->R > CP_MAX_R) return 0;
  std::unique_ptr<MG> mg(new MG());  // large struct: on the heap, one per call (reentrant)
  if (!mg->plan(*s, *p)) return 0;
  Arena a;
  return mg->layout(a);
}

int cp_mg_solve(const cp_shape *s, const double *Z, double *const *A, const double *const *T,
                const double *const *A_fmg, const cp_mg_params *prm, double *report, double *trace,
                void *ws, size_t ws_bytes, cp_stream_t stream) {
  if (!s || !Z || !A || !T || !prm || !report || !ws) return CP_EINVAL;
  if (s->N < 2 || s->N > CP_MAX_N || s->R < 1 || s->R > CP_MAX_R) return CP_EINVAL;
  if (prm->use_fmg && !A_fmg) return CP_EINVAL;
  // all driver state lives in this call's MG (heap) and the caller's workspace: two solves may
  // run concurrently (different workspaces, streams or devices)
  std::unique_ptr<MG> mgp(new MG());
  MG &mg = *mgp;
  struct EvGuard {
    MG &m;
    ~EvGuard() { m.destroy_events(); }
  } evguard{mg};
  if (!mg.plan(*s, *prm)) return CP_EINVAL;
  {
    Arena dry;
    const size_t need = mg.layout(dry);
    if (need == 0) return CP_EINVAL;
    if (ws_bytes < need) return CP_EWORKSPACE;
  }
  Arena a;
  a.base = static_cast<char *>(ws);
  a.cap = ws_bytes;
  a.dry = false;
  mg.layout(a);
  // the legacy default stream cannot be captured: run the solve on a private blocking stream
  // (implicitly ordered with the legacy stream), where the solve phase replays each FAS V-cycle
  // as one CUDA graph (CP_MG_GRAPH=0: plain launches).  Same kernels, same order: bitwise equal.
  struct Own {
    cudaStream_t s = nullptr;
    cudaGraphExec_t g = nullptr;
    void drop() {
      if (g) cudaGraphExecDestroy(g);
      g = nullptr;
    }
    ~Own() {
      drop();
      if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    }
  } own;
  mg.st = reinterpret_cast<cudaStream_t>(stream);
  if (mg.st == nullptr && cudaStreamCreate(&own.s) == cudaSuccess) {
    mg.st = own.s;
    stream = reinterpret_cast<cp_stream_t>(own.s);
  }
  mg.cst = stream;
  const bool want_graph = path_flag("CP_MG_GRAPH", 1) != 0 && mg.st != nullptr;
  bool captured = false;
  // one FAS V-cycle from the finest level (Algorithm 2), replayed from a graph when possible
  auto v_cycle = [&]() {
    if (want_graph && !captured && mg.err == CP_OK) {
      captured = true;
      cudaGraph_t graph = nullptr;
      if (cudaStreamBeginCapture(mg.st, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
        mg.fas_cycle(0, nullptr);
        const cudaError_t ec = cudaStreamEndCapture(mg.st, &graph);
        if (mg.err == CP_OK && ec == cudaSuccess && graph != nullptr &&
            cudaGraphInstantiate(&own.g, graph, 0) != cudaSuccess)
          own.g = nullptr;
        if (graph != nullptr) cudaGraphDestroy(graph);
        cudaGetLastError();  // a failed capture falls back to plain launches
        if (mg.err != CP_OK) {
          mg.err = CP_OK;
          own.drop();
        }
      }
    }
    if (own.g != nullptr) {
      if (cudaGraphLaunch(own.g, mg.st) != cudaSuccess) mg.err = CP_ECUDA;
    } else {
      mg.fas_cycle(0, nullptr);
    }
  };
  const int N = s->N, R = s->R;
  for (int k = 0; k < 16; ++k) report[k] = 0.0;
  const auto t0 = std::chrono::steady_clock::now();
  Level &f = mg.lv[0];
  f.Z = Z;
  for (int n = 0; n < N; ++n) f.A[n] = A[n];
  for (int l = 0; l < mg.L; ++l)
    for (int t = 0; t < mg.nt; ++t)
      if (l == 0)
        for (int n = 0; n < N; ++n) mg.copy(f.T[t][n], T[t * N + n], (size_t)s->dims[n] * R);
  cp_shape s1 = *s;
  s1.R = 1;
  mg.ok(cp_norm2(&s1, Z, f.nz2, mg.ws, mg.ws_bytes, stream));
  if (cudaMemsetAsync(mg.out_slots, 0, (size_t)4 * kOutSlots * 8, mg.st) != cudaSuccess) mg.err = CP_ECUDA;

  int ntrace = 0, cycles = 0, setup_cycles = 0, solve_cycles = 0, rebuilds = 0;
  auto record = [&](int phase, int cyc, double g) {
    if (trace && ntrace < prm->max_trace) {
      trace[4 * ntrace + 0] = phase;
      trace[4 * ntrace + 1] = cyc;
      trace[4 * ntrace + 2] = g;
      trace[4 * ntrace + 3] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      ++ntrace;
    }
  };
  double g = mg.fit(0, f.A, nullptr);
  bool converged = g < prm->tol;
  // setup phase
  double g_old = g;
  for (int cyc = 1; !converged && cyc <= prm->max_setup_cycles && mg.err == CP_OK; ++cyc) {
    mg.setup_cycle(0, cyc == 1, true);
    const double gn = mg.fit(0, f.A, nullptr);
    ++cycles;
    ++setup_cycles;
    record(0, cycles, gn);
    g = gn;
    if (!(gn >= prm->tol)) {
      converged = !(gn != gn) && gn < prm->tol;
      break;
    }
    if (cyc >= prm->min_setup_cycles && gn > (1.0 - prm->stagnation_eps) * g_old) break;
    g_old = gn;
  }
  // "Multilevel + FMG": one FMG-CP-FAS cycle computes a new approximation to the boot
  // factors, then the transfer operators are rebuilt by one down-sweep of CP-AMG-mult (boot
  // factors not updated).  fmg_guard = 1 selects reading R29 instead (not the paper's default):
  // the FMG result is kept only if it lowers g, else the setup iterate is restored and the
  // operators are not rebuilt.
  if (!converged && prm->use_fmg && mg.err == CP_OK) {
    for (int n = 0; n < N; ++n) mg.copy(f.prev[n], f.A[n], (size_t)s->dims[n] * R);
    mg.fmg(A_fmg);
    const double gf = mg.fit(0, f.A, nullptr);
    ++cycles;
    record(1, cycles, gf);
    if (prm->fmg_guard && !(gf < g)) {
      for (int n = 0; n < N; ++n) mg.copy(f.A[n], f.prev[n], (size_t)s->dims[n] * R);
    } else {
      g = gf;
      converged = g < prm->tol;
      if (!converged) mg.setup_cycle(0, false, false);
    }
  }
  // solve phase
  bool rebuilt = false;
  g_old = g;
  while (!converged && cycles < prm->max_cycles && mg.err == CP_OK) {
    for (int n = 0; n < N; ++n) mg.copy(f.prev[n], f.A[n], (size_t)s->dims[n] * R);
    v_cycle();
    double gn = mg.fit(0, f.A, nullptr);
    ++cycles;
    ++solve_cycles;
    record(2, cycles, gn);
    if (gn != gn) break;
    if (gn < prm->tol) {
      g = gn;
      converged = true;
      break;
    }
    if (solve_cycles > prm->solve_stagnation_after && gn >= g_old && !rebuilt) {
      for (int n = 0; n < N; ++n) mg.copy(f.A[n], f.prev[n], (size_t)s->dims[n] * R);
      mg.setup_cycle(0, false, false);
      own.drop();  // (re-captured after the rebuild)
      captured = false;
      rebuilt = true;
      ++rebuilds;
      gn = g_old;
    }
    g = gn;
    g_old = gn;
  }
  const double fval = (mg.err == CP_OK) ? mg.h_fit[0] : NAN;
  cudaStreamSynchronize(mg.st);
  report[0] = g;
  report[1] = fval;
  report[2] = cycles;
  report[3] = setup_cycles;
  report[4] = solve_cycles;
  report[5] = mg.L;
  report[6] = (mg.err != CP_OK) ? (double)mg.err : (converged ? 0.0 : 1.0);
  report[7] = ntrace;
  report[8] = rebuilds;
  report[9] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  report[10] = mg.fit_seconds;
  report[11] = mg.failed_mode;
  return (mg.err == CP_ENOTSPD) ? CP_OK : mg.err;
}

// cp_als_solve's own region after the sweep workspace: ||Z||^2, the fit output and one out word
// per sweep slot (a sweep k writes slot k mod kAlsSlots; every slot written since the last check
// is read back with g)
constexpr int kAlsSlots = 256;
constexpr size_t kAlsSmall = 64 + 4 * kAlsSlots;  // doubles

size_t cp_als_solve_workspace_bytes(const cp_shape *s) {
  const size_t w = cp_workspace_bytes(s);
  return w == 0 ? 0 : w + kAlsSmall * sizeof(double);
}

int cp_als_solve(const cp_shape *s, const double *Z, double *const *A, double tol, int32_t max_iters,
                 int32_t check_every, double *report, void *ws, size_t ws_bytes, cp_stream_t stream) {
  if (!s || !Z || !A || !report || !ws || check_every < 1 || max_iters < 1) return CP_EINVAL;
  const size_t w = cp_workspace_bytes(s);
  if (w == 0) return CP_EINVAL;
  if (ws_bytes < w + kAlsSmall * sizeof(double)) return CP_EWORKSPACE;
  // the legacy default stream cannot be captured: run the solve on a private blocking stream
  // (implicitly ordered with the legacy stream) and graph-capture there
  struct Own {
    cudaStream_t s = nullptr;
    cudaGraphExec_t g = nullptr;
    ~Own() {
      if (g) cudaGraphExecDestroy(g);
      if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    }
  } own;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (st == nullptr && cudaStreamCreate(&own.s) == cudaSuccess) {
    st = own.s;
    stream = reinterpret_cast<cp_stream_t>(st);
  }
  double *small = reinterpret_cast<double *>(static_cast<char *>(ws) + w);
  double *nz2 = small, *fitout = small + 16, *slots = small + 64;
  const auto t0 = std::chrono::steady_clock::now();
  double fit_s = 0.0;
  cp_shape s1 = *s;
  s1.R = 1;
  int rc = cp_norm2(&s1, Z, nz2, ws, w, stream);
  if (rc) return rc;
  if (cudaMemsetAsync(slots, 0, 4 * kAlsSlots * sizeof(double), st) != cudaSuccess) return CP_ECUDA;
  const int nslots = check_every < kAlsSlots ? check_every : kAlsSlots;
  std::vector<double> h(2 + s->N), hs((size_t)4 * nslots);
  double g = NAN;
  int it = 0, status = 1, failed_mode = -1;
  // one sweep (+ normalization) into out slot k
  auto sweep = [&](int k) -> int {
    int r = cp_als_sweep(s, Z, nz2, A, nullptr, slots + 4 * (k % kAlsSlots), ws, w, stream);
    if (r == CP_OK) r = cp_normalize_sort(s, A, 0, nullptr, ws, w, stream);
    return r;
  };
  // The check_every sweeps (+ normalization) between two stopping tests are captured once into
  // a CUDA graph and replayed: for small tensors the loop is launch-bound (~10 launches per
  // sweep).  Same kernels in the same order -- results are bitwise those of the plain loop.
  // Needs a capturable stream (not the legacy default stream); CP_ALS_GRAPH=0 disables.
  cudaGraphExec_t &gexec = own.g;
  {
    const bool want = path_flag("CP_ALS_GRAPH", 1) != 0 && st != nullptr && check_every > 1;
    if (want) {
      cudaGraph_t graph = nullptr;
      bool okc = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
      for (int k = 0; okc && k < check_every; ++k) okc = sweep(k) == CP_OK;
      const cudaError_t ec = cudaStreamEndCapture(st, &graph);
      if (okc && ec == cudaSuccess && graph != nullptr &&
          cudaGraphInstantiate(&gexec, graph, 0) != cudaSuccess)
        gexec = nullptr;
      if (graph != nullptr) cudaGraphDestroy(graph);
      cudaGetLastError();  // a failed capture falls back to the plain loop
      if (!okc) gexec = nullptr;
    }
  }
  for (it = 1; it <= max_iters; ++it) {
    if (gexec != nullptr && it % check_every == 1 && it + check_every - 1 <= max_iters) {
      if (cudaGraphLaunch(gexec, st) != cudaSuccess) return CP_ECUDA;
      it += check_every - 1;  // the graph ran sweeps it .. it + check_every - 1
    } else {
      if ((rc = sweep((it - 1) % check_every))) return rc;
    }
    if (it % check_every == 0 || it == max_iters) {
      const auto tf = std::chrono::steady_clock::now();
      if ((rc = cp_gradient(s, Z, nz2, A, nullptr, fitout, nullptr, ws, w, stream))) return rc;
      if (cudaMemcpyAsync(h.data(), fitout, (2 + s->N) * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
          cudaMemcpyAsync(hs.data(), slots, hs.size() * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
          cudaStreamSynchronize(st) != cudaSuccess)
        return CP_ECUDA;
      fit_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - tf).count();
      g = h[1];
      for (int k = 0; k < nslots; ++k)
        if (hs[4 * k + 2] != 0.0) {
          status = CP_ENOTSPD;
          failed_mode = (int)hs[4 * k + 3];
        }
      if (status == CP_ENOTSPD || g != g) {
        status = CP_ENOTSPD;
        break;
      }
      if (g < tol) {
        status = 0;
        break;
      }
    }
  }
  if ((rc = cp_normalize_sort(s, A, 1, nullptr, ws, w, stream))) return rc;
  cudaStreamSynchronize(st);
  report[0] = g;
  report[1] = h[0];
  report[2] = (it > max_iters) ? max_iters : it;
  report[3] = status;
  report[4] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  report[5] = fit_s;
  report[6] = failed_mode;
  return CP_OK;
}

}  // extern "C"
