"""Host time per call of cp_mttkrp: through the Python binding, and the bare C call with the
ctypes arguments built once (the library's own host cost: plan lookup, tensor-map encoding,
launch).   python tools/host_overhead.py c3 [mode]"""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpsynth  # noqa: E402
import paper_1111_6091_b200 as cp  # noqa: E402
from paper_1111_6091_b200 import _ptr, _ptr_array, _shape, _stream, colmajor, empty_factor, lib  # noqa: E402

name = sys.argv[1]
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 1
_, dims, R, *_ = cpsynth.CONFIGS[name]
Z = torch.randn(tuple(reversed(dims)), dtype=torch.float64, device="cuda")
A = [colmajor(torch.randn(I, R, dtype=torch.float64, device="cuda")) for I in dims]
ws = cp.Workspace(dims, R)
M = empty_factor(dims[mode], R, "cuda")
sh = ctypes.byref(_shape(dims, R))
args = (sh, _ptr(Z), _ptr_array([a if k != mode else None for k, a in enumerate(A)]), ctypes.c_int32(mode),
        _ptr(M), _ptr(ws.buf), ctypes.c_size_t(ws.nbytes), _stream(None))
f = lib().cp_mttkrp
for _ in range(10):
    cp.mttkrp(Z, dims, A, mode, M=M, ws=ws)
    f(*args)
torch.cuda.synchronize()
n = 300
res = {}
for label, fn in (("binding", lambda: cp.mttkrp(Z, dims, A, mode, M=M, ws=ws)), ("bare C call", lambda: f(*args))):
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    res[label] = (t1 - t0) / n * 1e6
print(f"{name} mode {mode}: host us/call " + ", ".join(f"{k} {v:.1f}" for k, v in res.items()))
