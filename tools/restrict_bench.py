import sys, os, torch
sys.path.insert(0, '.')
import cpsynth, paper_1111_6091_b200 as cp
dims = (512, 512, 512)
Z = torch.randn(512, 512, 512, dtype=torch.float64, device='cuda')
X = torch.empty(256, 512, 512, dtype=torch.float64, device='cuda')
ws = torch.empty(1 << 16, dtype=torch.uint8, device='cuda')
for n in range(3):
    wl, wr = cpsynth.transfer_weights(512, seed=n)
    wl, wr = torch.from_numpy(wl).cuda(), torch.from_numpy(wr).cuda()
    nd = list(dims); nd[n] = 256
    Xn = X.view(tuple(reversed(nd)))
    for _ in range(3): cp.restrict_structured(Z, dims, n, wl, wr, X=Xn, ws=ws)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): cp.restrict_structured(Z, dims, n, wl, wr, X=Xn, ws=ws)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(os.environ.get("CP_RESTRICT_BLOCK", "128"), "mode", n, f"{ms:.4f} ms", f"{1.5 * 2**30 / ms / 1e6:.0f} GB/s")
