"""Reference point for 2:1 read:write HBM streams (torch elementwise add, 1 GiB read, 0.5 GiB
written) -- the ceiling the structured restriction is compared against."""
import torch
Z = torch.randn(512, 512, 512, dtype=torch.float64, device='cuda')
X = torch.empty(512, 512, 256, dtype=torch.float64, device='cuda')
a, b = Z[:256], Z[256:]
Xv = X.view(256, 512, 512)
for _ in range(3):
    torch.add(a, b, out=Xv)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    torch.add(a, b, out=Xv)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"torch add 2:1 read:write: {ms:.4f} ms, {1.5 * 2**30 / ms / 1e6:.0f} GB/s")
Y = torch.empty_like(Z)
for _ in range(3): Y.copy_(Z)
torch.cuda.synchronize(); e0.record()
for _ in range(20): Y.copy_(Z)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"torch copy 1:1: {ms:.4f} ms, {2 * 2**30 / ms / 1e6:.0f} GB/s")
