set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for r in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --no-max-context --no-e2e --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()}, d['clocks']['reasons'])"
done
timeout 300 python tools/trace_kernel.py --kernel bq --cta-table > gpurun_out/trace_bq2.txt 2>&1
