# medium fused sweep: ms per 50 sweeps vs elements per CTA (CP_MEDIUM_ELEMS) on 50^3 R3 and 100^3 R5
for el in 3072 6144 12288; do
  for sz in "50 3" "100 5"; do
    echo "elems=$el size=$sz :: $(CP_MEDIUM_ELEMS=$el python - $sz <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import cpsynth, paper_1111_6091_b200 as cp
os.environ['CP_MEDIUM_SWEEP'] = '1'
s, R = int(sys.argv[1]), int(sys.argv[2]); dims = (s, s, s)
Z, A = cpsynth.random_problem(dims, R, seed=1)
Zd = torch.from_numpy(Z).cuda(); Ad = [torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t() for a in A]
nz = cp.norm2(Zd, dims)
cp.als_sweep(Zd, dims, Ad, nz, nsweeps=50); torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
e[0].record(); cp.als_sweep(Zd, dims, Ad, nz, nsweeps=50); e[1].record(); torch.cuda.synchronize()
print(f"{e[0].elapsed_time(e[1]) / 50 * 1e3:.1f} us/sweep")
PY
)"
  done
done
