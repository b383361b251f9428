# HEAD evidence (tests, smoke, bench, reference arm, launch list) + A/B of the c4a sweep against the round-1 tree (alt/r01)
bash tools/gpu_check.sh > gpurun_out/gpu_check.out 2>&1
for i in 1 2; do
  (cd alt/r01 && timeout 300 python bench.py --no-rows --no-cpu --steps 200 --warmup 10) > gpurun_out/ab_r01_$i.json 2> gpurun_out/ab_r01_$i.err
  timeout 300 python bench.py --no-rows --no-cpu --steps 200 --warmup 10 > gpurun_out/ab_head_$i.json 2> gpurun_out/ab_head_$i.err
done
tail -3 gpurun_out/pytest_gpu.log
python - <<'P'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])
    except Exception as e: print(f, 'ERR', e)
P
