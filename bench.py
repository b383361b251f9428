#!/usr/bin/env python
"""bench.py -- the hot path of arXiv 1111.6091 on B200: ALS sweeps/s on BASELINE.json's
largest single-GPU config (c4a: 3-way 512^3 fp64, R = 16, 1 GiB tensor).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c4a]

One step = one cp_als_sweep (per-mode MTTKRP, Gram/Hadamard,
Cholesky solve, functional f) on the device-resident tensor.  Rows a0 (||Z||^2, once per
tensor), a7 (restriction Z x_1 Phat^T, once per setup cycle) and a8 (cp_fit, the stopping
test the paper excludes from its timings) are timed in the same run and reported under
"rows".  Rank 0 prints ONE JSON line.  Multi-GPU: independent replicas (weak scaling; the
path has no exchange step at one tensor per GPU -- DESIGN.md "Multi-GPU").

--impl reference times the CPU oracle (oracle/, plain C fp64) on the same config and metric:
each step is a bounded sample (MTTKRP of a contiguous 1/16 of the output rows of every mode,
scaled to sweeps/s).
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import cpsynth  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback
PEAKS_LIB = os.path.join(ROOT, "paper_1111_6091_b200", "lib", "libcppeaks.so")


def fp64_peaks():
    """DFMA and DMMA TFLOP/s measured in THIS run (libcppeaks.so, include/cp_peaks.h): the fp64
    roofline denominators MEASURED_PEAKS.json lacks."""
    import ctypes
    L = ctypes.CDLL(PEAKS_LIB)
    a, b = ctypes.c_double(), ctypes.c_double()
    rc = L.cpp_fp64_peaks(ctypes.byref(a), ctypes.byref(b), 5)
    if rc != 0:
        raise RuntimeError(f"cpp_fp64_peaks failed ({rc})")
    return {"dfma_tflops": a.value, "dmma_tflops": b.value,
            "source": "libcppeaks.so in this run: best of 5 event-timed launches, 8 CTAs x 256 threads per SM "
                      "(DFMA: 8 independent fma chains/thread; DMMA: mma.sync m8n8k4 f64, 8 accumulators/warp)"}


def launch_floor_us():
    import ctypes
    L = ctypes.CDLL(PEAKS_LIB)
    u = ctypes.c_double()
    if L.cpp_launch_floor_us(2000, ctypes.byref(u)) != 0:
        return None
    return u.value


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4a", choices=list(cpsynth.CONFIGS))
    ap.add_argument("--no-rows", action="store_true", help="skip the per-row extra timings")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def max_over_ranks(ms, world, device):
    """Max of a per-rank duration over all ranks (the timing rule: device time, max over ranks);
    device = the process group's tensor device (cuda for nccl, cpu for gloo)."""
    if world <= 1:
        return float(ms)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_value(world, steps, t_max_ms):
    """Whole-job throughput: units all ranks processed / the slowest rank's time (weak scaling:
    every rank runs its own replica of the workload)."""
    return world * steps / (t_max_ms / 1000.0)


def metric_name(workload):
    _, dims, R, *_ = cpsynth.CONFIGS[workload]
    shape = "x".join(str(d) for d in dims)
    return f"ALS sweeps/s (fp64 {shape}, R={R}; MTTKRP HBM GB/s in roofline)"


def config_block(workload, world):
    idx, dims, R, C, l1, l2, note = cpsynth.CONFIGS[workload]
    P = int(np.prod(dims))
    return {"workload": workload, "desc": note, "dims": list(dims), "R": R, "congruence": C,
            "noise_l1": l1, "noise_l2": l2, "tensor_bytes": 8 * P,
            "step": "one ALS sweep (all N modes: MTTKRP + Gram/Hadamard + Cholesky solve + f; "
                    "dimension-tree: 2 passes over Z); K steps = one cp_als_sweeps(nsweeps=K) call "
                    "(L2-resident configs: K single-sweep calls, each timed alone after an L2 flush)",
            "l2_policy": ("inputs larger than L2 (no flush)" if 8 * P > 2 * 126 * 2**20
                          else "L2 flushed (256 MiB write) between timed steps"),
            "parallelism": f"replicas x{world}"}


# ---------------------------------------------------------------------------- clocks (NVML)
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def report(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------- oracle timing
def oracle_sampled_sweeps_per_s(d, min_seconds, max_steps=None, frac_den=16):
    """Time the CPU oracle on a bounded sample: per step, MTTKRP of a contiguous 1/frac_den of
    the output rows of every mode (each row of mode n costs the same P/I_n * R work), i.e.
    1/frac_den of a sweep's MTTKRP work (the R x R solves, < 0.1% of it, are not timed)."""
    import oracle
    dims, Z, A = d["dims"], d["Z"], d["A0"]
    t_total, sweeps, steps = 0.0, 0.0, 0
    while True:
        t0 = time.perf_counter()
        frac = 0.0
        for n in range(len(dims)):
            nr = max(1, dims[n] // frac_den)
            lo = (steps * nr) % max(1, dims[n] - nr + 1)
            oracle.mttkrp(Z, dims, A, n, rows=(lo, lo + nr))
            frac += nr / dims[n] / len(dims)
        t_total += time.perf_counter() - t0
        sweeps += frac
        steps += 1
        if (max_steps is not None and steps >= max_steps) or (max_steps is None and t_total >= min_seconds):
            break
    return sweeps / t_total, steps, t_total


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import oracle
    d = cpsynth.make_config(args.workload, with_transfer=False)
    cores = oracle.num_threads()
    for _ in range(args.warmup):
        oracle_sampled_sweeps_per_s(d, 0, max_steps=1)
    val, steps, t = oracle_sampled_sweeps_per_s(d, 0, max_steps=args.steps)
    sample = (f"oracle (plain C fp64, OpenMP over output rows) MTTKRP of a contiguous 1/16 of the "
              f"output rows of every mode per step, {steps} steps in {t:.2f} s, scaled to sweeps/s")
    line = {"impl": "reference", "metric": metric_name(args.workload), "value": val,
            "unit": "sweeps/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * t / steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE.json config recipe)",
            "config": config_block(args.workload, 1),
            "cpu_baseline": {"value": val, "unit": "sweeps/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": val, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- our arm
def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    import paper_1111_6091_b200 as cp
    from paper_1111_6091_b200 import colmajor

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    d = cpsynth.make_config(args.workload)
    dims, R = d["dims"], d["R"]
    P = int(np.prod(dims))
    Zh = torch.from_numpy(d["Z"]).pin_memory()
    Zd = Zh.to(dev, non_blocking=False)
    A0 = [torch.from_numpy(np.ascontiguousarray(a.T)).to(dev).t() for a in d["A0"]]
    A = [colmajor(a.clone()) for a in A0]
    for a, a0 in zip(A, A0):
        a.copy_(a0)
    ws = cp.Workspace(dims, R, dev)
    nz = cp.norm2(Zd, dims, ws=ws)
    out = torch.empty(4, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up (untimed)
    for _ in range(max(3, args.warmup)):
        cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws)
    torch.cuda.synchronize()
    for a, a0 in zip(A, A0):
        a.copy_(a0)

    # ---- timed region: K sweeps, device-timed with CUDA events on the launch stream
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    flush = None
    if 8 * P <= 2 * 126 * 2**20:
        # tensor fits in L2: time every step separately and overwrite L2 between steps
        flush = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]

    def timed_loop():
        n = 0
        if flush is None:
            # K consecutive sweeps = one cp_als_sweeps(nsweeps = K) call: an ALS loop on the
            # device-resident tensor; sweeps 2..K run steady-state (the previous sweep's At copies
            # and Gram totals, no prep launch -- capi.cu sweep_impl)
            e0.record(stream)
            cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws, nsweeps=args.steps)
            n += cp.last_launch_count()
            e1.record(stream)
        else:
            for k in range(args.steps):
                flush.zero_()
                evs[k][0].record(stream)
                cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws)
                n += cp.last_launch_count()
                evs[k][1].record(stream)
        torch.cuda.synchronize()
        return (e0.elapsed_time(e1) if flush is None else sum(a.elapsed_time(b) for a, b in evs)), n

    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    with sampler:
        ms, launches = timed_loop()
    barrier()
    # the roofline's per-launch durations: a second K-step loop with CUDA events around every
    # streaming-kernel launch (cp_profile_*).  Kept out of the headline loop: an event between
    # two launches serializes them (no programmatic dependent launch), ~10 us per sweep on c4a.
    cp.profile_enable(True)
    ms_prof, _ = timed_loop()
    nlaunch_prof, prof_ms, prof_bytes = cp.profile_read()
    cp.profile_enable(False)
    barrier()
    res = out.cpu().numpy()
    if res[2] != 0 or not math.isfinite(res[0]):
        raise SystemExit(f"sweep failed: status {res[2]} mode {res[3]} f {res[0]}")
    t_max = max_over_ranks(ms, world, dev)
    value = job_value(world, args.steps, t_max)

    # ---- roofline of the dominant kernel (the Z-streaming MTTKRP kernel)
    peaks = json.load(open(PEAKS_PATH)) if os.path.exists(PEAKS_PATH) else {}
    peak = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs, STREAM copy)" if peak else "fallback (B200_PROFILING.md)"
    peak = peak or FALLBACK_HBM
    avg_ms = prof_ms / max(1, nlaunch_prof)
    bytes_per_launch = prof_bytes / max(1, nlaunch_prof)
    achieved = bytes_per_launch / (avg_ms / 1000.0) / 1e9 if nlaunch_prof else None
    traffic = None
    if os.path.exists(TRAFFIC_PATH):
        tr = json.load(open(TRAFFIC_PATH)).get(args.workload)
        if tr:
            traffic = tr.get("dram_bytes_per_launch")
    peaks64 = fp64_peaks()
    # the FP64 tensor pipe the consumers run on (DMMA, mma.sync m8n8k4): 2 x (8 NT) flops per Z element
    # per launch (ranks padded to the n-tiles of 8), against the DMMA peak measured in this run;
    # the DFMA pipe is idle in these kernels (ncu: sm__inst_executed_pipe_fp64 ~1 %)
    rpad = 8 * ((R + 7) // 8)
    dmma_tf = (2.0 * rpad * P) / (avg_ms / 1000.0) / 1e12 if nlaunch_prof else None
    roofline = {"kernel": "stream_mma_kernel (the two Z passes of the dimension-tree sweep, FP64 "
                          "tensor-core consumers: Y_L pass + mode-2 MTTKRP pass)", "bound": "hbm",
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "peak_source": peak_src, "alg_bytes_per_launch": bytes_per_launch,
                "avg_launch_ms": avg_ms, "launches_timed": nlaunch_prof,
                "share_of_step": (prof_ms / ms_prof) if ms_prof > 0 else None,
                "timed_region": "a second K-step loop of the same sweep with CUDA events around every "
                                "streaming-kernel launch (the headline loop runs without them)",
                "frac_of_8TBs_nominal": (achieved / 8000.0) if achieved else None,
                "pipes": {"fp64_tensor_dmma": {"achieved_tflops": dmma_tf, "peak_tflops": peaks64["dmma_tflops"],
                                               "frac": dmma_tf / peaks64["dmma_tflops"] if dmma_tf else None,
                                               "work": f"2 x {rpad} (ranks padded to n-tiles of 8) flops per Z element"},
                          "fp64_dfma": {"peak_tflops": peaks64["dfma_tflops"],
                                        "note": "not used by this kernel (DMMA consumers); ncu pipe_fp64 ~1 %"},
                          "hbm_frac": (achieved / peak) if achieved else None},
                "fp64_peaks": peaks64}
    # the whole step against the same peak: the sweep's algorithmic bytes (every streaming launch
    # of one sweep, as counted for the kernel above) at the copy peak vs the measured step time
    step_bytes = prof_bytes / max(1, args.steps) if nlaunch_prof < 8192 else float("nan")  # (cp.h: 8192 recorded launches)
    step_ms = t_max / args.steps
    roofline["step"] = {"alg_bytes": step_bytes, "bound_ms": step_bytes / (peak * 1e9) * 1e3,
                        "frac": (step_bytes / (peak * 1e9) * 1e3) / step_ms if step_ms > 0 else None,
                        "note": "sweeps/s as a fraction of its HBM roofline (all N modes' Z passes at the peak)"}

    # ---- extra rows (same run, outside the timed region)
    rows = {}
    if not args.no_rows:
        rows = time_rows(cp, torch, d, Zd, A, nz, ws, dev, stream, dims, R, P, peaks64)

    # ---- e2e through the public API with host buffers
    e2e = time_e2e(cp, torch, d, Zh, Zd, A0, A, nz, ws, dev, stream, dims, R, P, min(args.steps, 10))

    line = {"metric": metric_name(args.workload), "value": value, "unit": "sweeps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE.json config recipe)",
            "config": config_block(args.workload, world), "roofline": roofline,
            "clocks": sampler.report(), "e2e": e2e, "gpu_launches": launches, "rows": rows,
            "f_after_timed_sweeps": float(res[0])}

    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle
        val, steps, t = oracle_sampled_sweeps_per_s(d, min_seconds=10.0)
        cores = oracle.num_threads()
        oracle.set_threads(1)
        val1, steps1, t1 = oracle_sampled_sweeps_per_s(d, min_seconds=5.0)
        oracle.set_threads(cores)
        line["cpu_baseline"] = {
            "value": val, "unit": "sweeps/s", "cores": cores, "kind": "oracle",
            "value_1_thread": val1, "sample_1_thread": f"{steps1} sample steps in {t1:.1f} s on one host core",
            "sample": (f"oracle MTTKRP of a contiguous 1/16 of the output rows of every mode per "
                       f"sample step, {steps} steps in {t:.1f} s on the host cores, scaled to sweeps/s "
                       f"(R x R solves not timed)"),
            "rows": oracle_rows(cores)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def oracle_rows(cores):
    """The oracle beside the GPU rows: the multigrid solve on c0-c2 (per cycle:
    the first cycles of each solve, c0 to the tolerance) and a dense restriction mode product
    (a 1/16 slab of the c3 shape, scaled), on the host cores."""
    import oracle
    from oracle import mg
    out = {"cores": cores}
    for name, coarsest, maxc in (("c0", 10, 500), ("c1", 0, 4), ("c2", 25, 3)):
        dc = cpsynth.make_config(name, with_transfer=False)
        dd, Rc = dc["dims"], dc["R"]
        T0 = [cpsynth.uniform_init(dd, Rc, seed=10 + t) for t in range(2)]
        t0 = time.perf_counter()
        _, rep, _ = mg.mg_solve(dc["Z"], dd, dc["A0"], T0, coarsest=coarsest, tol=1e-9, max_cycles=maxc)
        dt = time.perf_counter() - t0
        out[f"mg_solve_{name}_ml"] = {"seconds": dt, "cycles": rep["cycles"], "status": rep["status"],
                                      "seconds_per_cycle": dt / max(1, rep["cycles"]),
                                      "note": "to g <= 1e-9" if maxc >= 500 else f"first {rep['cycles']} cycles only (setup cycles run in full)"}
    Z = np.random.default_rng(1).standard_normal((16, 256, 256))  # 1/16 slab of 256^3 (mode-3 planes)
    U = np.asfortranarray(np.random.default_rng(2).standard_normal((128, 256)))
    t0 = time.perf_counter()
    oracle.mode_product(Z, (256, 256, 16), 0, U)
    dt = time.perf_counter() - t0
    out["restriction_c3_dense_mode0"] = {"seconds_full_scaled": 16 * dt,
                                         "GFLOPs": 2.0 * 128 * 256 * 256 * 16 / dt / 1e9,
                                         "sample": "Z x_1 U, U 128 x 256, on a 256 x 256 x 16 slab, x16"}
    return out


def time_rows(cp, torch, d, Zd, A, nz, ws, dev, stream, dims, R, P, peaks64):
    rows = {}
    reps = 20
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def timed(fn, n=reps):
        fn()
        torch.cuda.synchronize()
        ev[0].record(stream)
        for _ in range(n):
            fn()
        ev[1].record(stream)
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / n

    # a1: MTTKRP per mode (cp_mttkrp: prep + stream + reduce)
    M = [torch.empty((R, I), dtype=torch.float64, device=dev).t() for I in dims]
    for n in range(len(dims)):
        t = timed(lambda: cp.mttkrp(Zd, dims, A, n, M=M[n], ws=ws))
        alg = 8.0 * (P + sum(dims[k] * R for k in range(len(dims)) if k != n) + dims[n] * R)
        rows[f"mttkrp_mode{n}"] = {"ms": t, "alg_GBps": alg / t / 1e6}
    # a0: ||Z||^2
    t = timed(lambda: cp.norm2(Zd, dims, ws=ws))
    rows["norm2"] = {"ms": t, "alg_GBps": 8.0 * P / t / 1e6}
    # a8: cp_fit (residual pass + N MTTKRPs + gradients)
    t = timed(lambda: cp.fit(Zd, dims, A, nz, ws=ws), n=5)
    rows["fit"] = {"ms": t}
    # NEXT-2: cp_gradient (all N gradients at one iterate through the dimension tree, no residual
    # pass; what the multigrid driver's stopping tests and FAS operators call)
    t = timed(lambda: cp.gradient(Zd, dims, A, nz, ws=ws), n=5)
    rows["gradient"] = {"ms": t, "z_passes": 2 if len(dims) >= 3 else len(dims),
                        "alg_GBps": 2 * 8.0 * P / t / 1e6 if len(dims) >= 3 else None}
    # a7: restriction Z x_1 Phat^T (dense orthonormal Phat, I_1 -> ceil(I_1/2))
    Ph = d["Phat"][0]
    U = torch.from_numpy(np.ascontiguousarray(Ph)).to(dev).t()  # (Ic x I1) column-major = Phat^T
    from paper_1111_6091_b200 import colmajor, empty_factor
    U = colmajor(U)
    J = U.shape[0]
    nd = list(dims)
    nd[0] = J
    X = torch.empty(tuple(reversed(nd)), dtype=torch.float64, device=dev)
    t = timed(lambda: cp.mode_product(Zd, dims, 0, U, X=X), n=3)
    flops = 2.0 * J * P
    rows["restriction_mode0"] = {"ms": t, "TFLOPs": flops / t / 1e9, "J": J,
                                 "alg_GBps": 8.0 * (P + P * J / dims[0]) / t / 1e6}
    del X
    # BASELINE.json configs[3]: restriction of a 256^3 tensor by a dense 256 x 128 transfer
    # operator, every mode (random data of that shape; fp64-compute-bound: DMMA roofline)
    Z3 = torch.randn(256, 256, 256, dtype=torch.float64, device=dev)
    for n in range(3):
        U3 = colmajor(torch.randn(128, 256, dtype=torch.float64, device=dev))
        nd3 = [256, 256, 256]
        nd3[n] = 128
        X3 = torch.empty(tuple(reversed(nd3)), dtype=torch.float64, device=dev)
        t = timed(lambda: cp.mode_product(Z3, (256, 256, 256), n, U3, X=X3), n=10)
        tf = 2.0 * 128 * 256**3 / t / 1e9
        rows[f"restriction_c3_dense_mode{n}"] = {"ms": t, "TFLOPs": tf,
                                                 "frac_dmma_peak": tf / peaks64["dmma_tflops"],
                                                 "peak_note": "DMMA peak measured in this run (libcppeaks.so)"}
        del X3
    del Z3
    # NEXT-3: the same restriction with the structured BAMG operator (cp_restrict_structured:
    # 3-tap gather + bidiagonal substitution per fiber; HBM-bound), every mode
    for n in range(len(dims)):
        wl, wr = cpsynth.transfer_weights(dims[n], seed=512 + n)
        wld, wrd = torch.from_numpy(wl).to(dev), torch.from_numpy(wr).to(dev)
        nd = list(dims)
        nd[n] = (dims[n] + 1) // 2
        X = torch.empty(tuple(reversed(nd)), dtype=torch.float64, device=dev)
        rws = torch.empty(32 * dims[n] + 64, dtype=torch.uint8, device=dev)
        t = timed(lambda: cp.restrict_structured(Zd, dims, n, wld, wrd, X=X, ws=rws), n=10)
        alg = 8.0 * (P + P * nd[n] / dims[n])
        rows[f"restriction_structured_mode{n}"] = {"ms": t, "alg_GBps": alg / t / 1e6,
                                                   "frac_hbm": alg / t / 1e6 / (json.load(open(PEAKS_PATH)).get("hbm_gbs", FALLBACK_HBM) if os.path.exists(PEAKS_PATH) else FALLBACK_HBM)}
        del X
    # BASELINE.json configs[3] (c3: 256^3, R = 8, 128 MiB ~ L2): the sweep and the MTTKRP of every
    # mode, L2 flushed (256 MiB write) before each rep and each rep timed by its own event pair
    if tuple(dims) != (256, 256, 256):
        d3, R3 = (256, 256, 256), 8
        P3 = 256 ** 3
        Z3 = torch.randn(d3, dtype=torch.float64, device=dev)
        A3 = [colmajor(torch.randn(I, R3, dtype=torch.float64, device=dev)) for I in d3]
        ws3 = cp.Workspace(d3, R3)
        nz3 = cp.norm2(Z3, d3, ws=ws3)
        out3 = torch.empty(4, dtype=torch.float64, device=dev)
        fl = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)

        def flushed(fn, n=20):
            fn()
            tot = 0.0
            for _ in range(n):
                fl.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fn()
                e1.record(stream)
                e1.synchronize()
                tot += e0.elapsed_time(e1)
            return tot / n

        t = flushed(lambda: cp.als_sweep(Z3, d3, A3, nz3, out=out3, ws=ws3))
        rows["c3_sweep"] = {"ms": t, "sweeps_per_s": 1e3 / t, "z_passes": 2,
                            "alg_GBps_2pass": 2 * 8.0 * P3 / t / 1e6, "l2": "flushed before each rep"}
        # the ALS loop itself: K sweeps in one cp_als_sweeps call (steady state: no prep launch, the
        # last mode solved inside the pass; Z = 128 MiB stays partly L2-resident between passes)
        cp.als_sweep(Z3, d3, A3, nz3, out=out3, ws=ws3, nsweeps=50)
        t = timed(lambda: cp.als_sweep(Z3, d3, A3, nz3, out=out3, ws=ws3, nsweeps=50), n=4) / 50
        rows["c3_sweep_steady"] = {"ms": t, "sweeps_per_s": 1e3 / t, "z_passes": 2,
                                   "alg_GBps_2pass": 2 * 8.0 * P3 / t / 1e6,
                                   "l2": "not flushed: one cp_als_sweeps(50) call, device-resident loop"}
        M3 = [empty_factor(I, R3, dev) for I in d3]
        for n in range(3):
            t = flushed(lambda: cp.mttkrp(Z3, d3, A3, n, M=M3[n], ws=ws3))
            alg = 8.0 * (P3 + sum(d3[k] * R3 for k in range(3) if k != n) + d3[n] * R3)
            rows[f"c3_mttkrp_mode{n}"] = {"ms": t, "alg_GBps": alg / t / 1e6, "l2": "flushed before each rep"}
        del Z3, A3, ws3, M3, fl
    # the 4-way roofline point of BASELINE.json configs[4] (c4b: 96^4, R = 10): the sweep (two
    # dimension-tree passes) and every MTTKRP, on device-random data (timing does not depend on
    # the values; the c4b parity tests use the config's own tensor)
    if tuple(dims) != (96, 96, 96, 96):
        d4, R4 = (96, 96, 96, 96), 10
        P4 = 96 ** 4
        Z4 = torch.randn(d4, dtype=torch.float64, device=dev)
        A4 = [colmajor(torch.randn(I, R4, dtype=torch.float64, device=dev)) for I in d4]
        ws4 = cp.Workspace(d4, R4)
        nz4 = cp.norm2(Z4, d4, ws=ws4)
        out4 = torch.empty(4, dtype=torch.float64, device=dev)
        t = timed(lambda: cp.als_sweep(Z4, d4, A4, nz4, out=out4, ws=ws4), n=20)
        rows["c4b_sweep"] = {"ms": t, "sweeps_per_s": 1e3 / t, "z_passes": 2,
                             "alg_GBps_2pass": 2 * 8.0 * P4 / t / 1e6}
        M4 = [empty_factor(I, R4, dev) for I in d4]
        for n in range(4):
            t = timed(lambda: cp.mttkrp(Z4, d4, A4, n, M=M4[n], ws=ws4))
            alg = 8.0 * (P4 + sum(d4[k] * R4 for k in range(4) if k != n) + d4[n] * R4)
            rows[f"c4b_mttkrp_mode{n}"] = {"ms": t, "alg_GBps": alg / t / 1e6}
        del Z4, A4, ws4, M4
    # 8(d): full multigrid solve time to a stated g tolerance on BASELINE.json configs c0 (2-level
    # cycle: coarsest 10), c1 (BAMG setup + FAS V-cycles to g <= 1e-9, coarsest 2R) and c2 (3 levels:
    # coarsest 25): ML, ML+FMG (the paper's P:492 combination) and ML+FMG with reading R29's
    # guard, beside the plain ALS solve to the same tolerance.  seconds include the stopping tests,
    # seconds_excl_stop excludes them (the paper excludes them).  A run that does not reach
    # the tolerance is reported as unsuccessful, as the paper counts them.
    try:
        import importlib.util
        spec = importlib.util.spec_from_file_location("mg_bench", os.path.join(ROOT, "tools", "mg_bench.py"))
        mgb = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mgb)
        for name, coarsest, mc in (("c0", 10, 500), ("c1", 0, 500), ("c2", 25, 200)):
            mgb.run(name, tol=1e-9, coarsest=coarsest, max_cycles=min(mc, 20), als=False)  # warm-up
            rows[f"mg_solve_{name}"] = mgb.run(name, tol=1e-9, coarsest=coarsest, max_cycles=mc)
        # the paper's own dense problem (Table 4 context: s = 50, R = 2)
        rows["mg_solve_dense50_R2"] = mgb.run("dense50", R=2, tol=1e-9)
        # s = 100, R = 3 (Table 4 context: ML+FMG 9 cycles): the case where the multigrid beats ALS
        mgb.run("dense100", R=3, tol=1e-10, max_cycles=20, als=False)  # warm-up (plans, graphs)
        rows["mg_solve_dense100_R3"] = mgb.run("dense100", R=3, tol=1e-10)
    except Exception as e:  # the row is informative; the sweep metric stands without it
        rows["mg_solve_error"] = {"error": repr(e)}
    # 8(d): c0-c2 are L2-resident and latency/launch-bound: microseconds per sweep (K sweeps captured
    # in one CUDA graph and replayed, device time by events) and the launch-floor fraction
    # (launches per sweep x the empty-kernel launch time of this run / the sweep time)
    floor = launch_floor_us()
    for name in ("c0", "c1", "c2"):
        dc = cpsynth.make_config(name, with_transfer=False)
        dd, Rc = dc["dims"], dc["R"]
        Zc = torch.from_numpy(dc["Z"]).to(dev)
        Ac = [colmajor(torch.from_numpy(np.ascontiguousarray(a)).to(dev)) for a in dc["A0"]]
        wsc = cp.Workspace(dd, Rc)
        nzc = cp.norm2(Zc, dd, ws=wsc)
        outc = torch.empty(4, dtype=torch.float64, device=dev)
        cp.als_sweep(Zc, dd, Ac, nzc, out=outc, ws=wsc)
        nl = cp.last_launch_count()
        K = 50
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(3):
                cp.als_sweep(Zc, dd, Ac, nzc, out=outc, ws=wsc, stream=side)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(K):
                cp.als_sweep(Zc, dd, Ac, nzc, out=outc, ws=wsc)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / (4 * K)
        # the same K sweeps as ONE cp_als_sweeps(K) call (steady-state sweeps)
        cp.als_sweep(Zc, dd, Ac, nzc, out=outc, ws=wsc, nsweeps=K)
        nls = cp.last_launch_count()
        us_steady = 1e3 * timed(lambda: cp.als_sweep(Zc, dd, Ac, nzc, out=outc, ws=wsc, nsweeps=K), n=4) / K
        rows[f"{name}_sweep_latency"] = {
            "us_per_sweep": us, "sweeps_per_s": 1e6 / us, "launches_per_sweep": nl,
            "us_per_sweep_one_call": us_steady, "launches_per_sweep_one_call": nls / K,
            "launch_floor_us": floor, "launch_floor_frac": (nl * floor / us) if floor else None,
            "path": "fused single-CTA kernel (small_sweep.cu)" if nl == 1 else "general dimension-tree sweep",
            "timing": f"{K} sweeps in one CUDA graph, 4 replays, L2-resident (no flush)"}
        del g, Zc, Ac, wsc
    # the same sweep with the DFMA streaming consumers (CP_STREAM_MMA=0: FP64 tensor cores only in
    # the mode products, as BASELINE.json's north star first proposed)
    os.environ["CP_STREAM_MMA"] = "0"
    try:
        ws2 = cp.Workspace(dims, R)
        A2 = [torch.empty((R, a.shape[0]), dtype=torch.float64, device=dev).t().copy_(a) for a in A]
        out2 = torch.empty(4, dtype=torch.float64, device=dev)
        t = timed(lambda: cp.als_sweep(Zd, dims, A2, nz, out=out2, ws=ws2))
        rows["sweep_dfma_consumers"] = {"ms": t}
        t = timed(lambda: cp.mttkrp(Zd, dims, A, len(dims) - 1, M=M[-1], ws=ws2))
        alg = 8.0 * (P + sum(dims[k] * R for k in range(len(dims) - 1)) + dims[-1] * R)
        rows[f"mttkrp_mode{len(dims) - 1}_dfma_consumers"] = {"ms": t, "alg_GBps": alg / t / 1e6}
        del ws2
    finally:
        del os.environ["CP_STREAM_MMA"]
    return rows


def time_e2e(cp, torch, d, Zh, Zd, A0, A, nz, ws, dev, stream, dims, R, P, K):
    """Same metric through the public API with host buffers: every step copies the tensor and
    the initial factors from pinned host memory, computes ||Z||^2, runs the sweep and reads f."""
    Ah = [torch.from_numpy(np.ascontiguousarray(a.T)).pin_memory() for a in d["A0"]]
    outh = torch.empty(4, dtype=torch.float64).pin_memory()
    Aout = [torch.empty_like(h).pin_memory() for h in Ah]
    out = torch.empty(4, dtype=torch.float64, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def step():
        Zd.copy_(Zh, non_blocking=True)
        for a, h in zip(A, Ah):
            a.t().copy_(h, non_blocking=True)
        cp.norm2(Zd, dims, out=nz, ws=ws)
        cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws)
        outh.copy_(out, non_blocking=True)
        for a, h in zip(A, Aout):
            h.copy_(a.t(), non_blocking=True)

    step()
    torch.cuda.synchronize()
    ev[0].record(stream)
    for _ in range(K):
        step()
    ev[1].record(stream)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    return {"value": K / (ms / 1000.0), "unit": "sweeps/s", "steps": K,
            "h2d_bytes_per_step": 8 * P + sum(8 * I * R for I in dims),
            "d2h_bytes_per_step": 32 + sum(8 * I * R for I in dims),
            "note": "per step: H2D of Z and the factors from pinned memory, cp_norm2, cp_als_sweep, D2H of "
                    "[f, f~, status, mode] and of the updated factors (the sweep's result)"}


if __name__ == "__main__":
    sys.exit(main())
