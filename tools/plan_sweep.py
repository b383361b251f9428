"""Sweep stream-kernel plan knobs (env overrides read by capi.cu) on the dimension-tree sweep.
Each setting runs in a fresh subprocess; prints ms/sweep and the streaming-kernel share.

    python tools/plan_sweep.py c4a "CP_STAGE_BYTES=20480,CP_RING_BYTES=98304" "CP_STAGE_BYTES=40960" ...
    python tools/plan_sweep.py --one c4a        (worker: one measurement with the current env)
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(name, sweeps=50):
    import numpy as np
    import torch
    sys.path.insert(0, HERE)
    import cpsynth
    import paper_1111_6091_b200 as cp
    _, dims, R, *_ = cpsynth.CONFIGS[name]
    rng = np.random.default_rng(0)
    Zd = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device="cuda")
    A = [torch.from_numpy(np.ascontiguousarray(rng.standard_normal((R, I)))).cuda().t() for I in dims]
    ws = cp.Workspace(dims, R)
    nz = cp.norm2(Zd, dims, ws=ws)
    out = torch.empty(4, dtype=torch.float64, device="cuda")
    for _ in range(5):
        cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(sweeps):
        cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws)
    ev[1].record()
    torch.cuda.synchronize()
    ms_plain = ev[0].elapsed_time(ev[1]) / sweeps
    cp.profile_enable(True)
    cp.profile_read()
    ev[0].record()
    for _ in range(sweeps):
        cp.als_sweep(Zd, dims, A, nz, out=out, ws=ws)
    ev[1].record()
    torch.cuda.synchronize()
    n, sms, b = cp.profile_read()
    cp.profile_enable(False)
    ms = ev[0].elapsed_time(ev[1]) / sweeps
    print(f"{ms_plain:.4f} ms/sweep ({ms:.4f} profiled)  stream {sms / sweeps:.4f} ms/sweep ({n // sweeps} launches, "
          f"{b / (sms * 1e6):.0f} GB/s alg)  status={out[2].item():.0f}")


if __name__ == "__main__":
    if sys.argv[1] == "--one":
        one(sys.argv[2])
        sys.exit(0)
    name = sys.argv[1]
    for cfg in sys.argv[2:]:
        env = dict(os.environ)
        if cfg != "-":
            for kv in cfg.split(","):
                k, v = kv.split("=")
                env[k] = v
        r = subprocess.run([sys.executable, __file__, "--one", name], env=env, capture_output=True, text=True)
        line = (r.stdout.strip().splitlines() or [r.stderr.strip()[-300:]])[-1]
        print(f"{name} {cfg:>48s} :: {line}", flush=True)
