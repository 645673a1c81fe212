# headline step and per-kernel times for several segment targets of the tcgen05 path (RACE_SEG_TARGET)
for t in 1184 888 592 444 296; do
  for r in 1 2; do
    RACE_SEG_TARGET=$t timeout 300 python bench.py --no-cpu-baseline --no-max-context --no-e2e --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()})"
  done
done
