"""Where a single cp_mttkrp call's time goes at one config: host time per call, device time of
back-to-back calls, of CUDA-graph replays, and of single calls after an L2 flush.
    python tools/mttkrp_overhead.py c3 [mode] [ENV=VAL,...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402
from paper_1111_6091_b200 import colmajor, empty_factor  # noqa: E402

name = sys.argv[1]
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for kv in (sys.argv[3].split(",") if len(sys.argv) > 3 else []):
    k, v = kv.split("=")
    os.environ[k] = v
_, dims, R, *_ = cpsynth.CONFIGS[name]
Z = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device="cuda")
A = [colmajor(torch.randn(I, R, dtype=torch.float64, device="cuda")) for I in dims]
ws = cp.Workspace(dims, R)
M = empty_factor(dims[mode], R, "cuda")
fl = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
fl2 = torch.ones(256 * 2**17, dtype=torch.float64, device="cuda")  # 256 MiB read after the write flush
call = lambda s=None: cp.mttkrp(Z, dims, A, mode, M=M, ws=ws, stream=s)  # noqa: E731
for _ in range(5):
    call()
torch.cuda.synchronize()
# host time per call (no sync; the queue absorbs the work)
n = 200
t0 = time.perf_counter()
for _ in range(n):
    call()
t1 = time.perf_counter()
torch.cuda.synchronize()
host_us = (t1 - t0) / n * 1e6
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
# back-to-back
e0, e1 = ev(), ev()
e0.record()
for _ in range(50):
    call()
e1.record()
e1.synchronize()
b2b = e0.elapsed_time(e1) / 50 * 1e3
# graph
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    call(s)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(20):
        call(torch.cuda.current_stream())
g.replay()
torch.cuda.synchronize()
e0, e1 = ev(), ev()
e0.record()
g.replay()
e1.record()
e1.synchronize()
gr = e0.elapsed_time(e1) / 20 * 1e3
# flushed single calls; and flushed single graph replays of one call
g1 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g1):
    call(torch.cuda.current_stream())
fs, fg, fc = [], [], []
for _ in range(20):
    fl.zero_()
    e0, e1 = ev(), ev()
    e0.record()
    call()
    e1.record()
    e1.synchronize()
    fs.append(e0.elapsed_time(e1) * 1e3)
    fl.zero_()
    e0, e1 = ev(), ev()
    e0.record()
    g1.replay()
    e1.record()
    e1.synchronize()
    fg.append(e0.elapsed_time(e1) * 1e3)
    # write flush, then a 256 MiB read: L2 cold AND clean (no dirty lines written back inside
    # the timed call)
    fl.zero_()
    fl2.sum()
    e0, e1 = ev(), ev()
    e0.record()
    g1.replay()
    e1.record()
    e1.synchronize()
    fc.append(e0.elapsed_time(e1) * 1e3)
print(f"{name} mode {mode} {sys.argv[3] if len(sys.argv) > 3 else ''}: host {host_us:.1f} us/call | back-to-back "
      f"{b2b:.1f} | graph {gr:.1f} | flushed call {np.median(fs):.1f} | flushed graph {np.median(fg):.1f} | "
      f"clean-cold graph {np.median(fc):.1f} us "
      f"({cp.last_launch_count()} launches)")
