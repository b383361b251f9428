# Round-1 session-2 evidence: default bench (+ reference arm), the ncu launch list of the bench
# command, and ncu --set full captures of the sweep kernels and the structured restriction,
# exported on the box as raw/details CSV (the .ncu-rep files are too large to bring back).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_bench_c4a.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-rows > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'stream_mma|ylsolve|solve_kernel|prep' --launch-skip 14 --launch-count 7 -f -o /tmp/r01d_sweep_c4a python tools/prof_sweep.py c4a 3 > gpurun_out/ncu_sweep.log 2>&1
cat > /tmp/rs.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import cpsynth, paper_1111_6091_b200 as cp
dims = (512, 512, 512)
Z = torch.randn(512, 512, 512, dtype=torch.float64, device='cuda')
for n in range(3):
    wl, wr = cpsynth.transfer_weights(512, seed=n)
    for _ in range(2):
        cp.restrict_structured(Z, dims, n, torch.from_numpy(wl).cuda(), torch.from_numpy(wr).cuda())
torch.cuda.synchronize()
PY
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'restrict_(inner|mode0)' -f -o /tmp/r01d_restrict_c4a python /tmp/rs.py > gpurun_out/ncu_restrict.log 2>&1
for r in r01d_sweep_c4a r01d_restrict_c4a; do
  ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>&1
  ncu -i /tmp/$r.ncu-rep --page details --csv > gpurun_out/$r.details.csv 2>&1
done
ls -la gpurun_out; du -sh gpurun_out
