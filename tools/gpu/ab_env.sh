# A/B of an environment switch on the headline step: bash tools/gpu/ab_env.sh VAR=value [rounds]
for r in $(seq ${2:-4}); do
  for e in "" "$1"; do
    env $e timeout 300 python bench.py --no-cpu-baseline --no-max-context --no-e2e --steps 50 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${e:-default}', round(d['ms_per_step']*1e3,1))"
  done
done
