# bench (default) + reference arm + ncu launch list of the default bench command
mkdir -p gpurun_out
T=${TAG:-r02d}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-rows > gpurun_out/${T}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_bench_c4a.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu --no-rows > gpurun_out/${T}_ncu_bench.log 2>&1
python - <<'PY'
import json,os
T=os.environ.get("TAG","r02d")
d=json.load(open(f"gpurun_out/{T}_bench.json"))
print({k:d[k] for k in ("value","ms_per_step","gpu_launches")}, d["roofline"]["frac"], d["roofline"]["step"]["frac"], d["clocks"])
PY
