for env in "CP_MG_STRUCTURED=1" "CP_MG_STRUCTURED=0"; do
  for prob in "dense50 2" "dense100 3"; do
  echo "== $env $prob"; env $env timeout 300 python tools/mg_bench.py $prob 1e-9 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: (v.get('seconds'), v.get('cycles', v.get('iterations')), v.get('g'), v.get('status')) for k, v in d.items() if isinstance(v, dict)})"
  done
done
