# quick GPU iteration: a parity subset, the causal bench (kernel times) and a trace of one kernel
# usage: bash tools/gpu/quick.sh "<pytest -k expr>" <trace kernel: fwd|bq|bk|none> [runs]
set -x
K="$1"; TK="${2:-none}"; RUNS="${3:-2}"
if [ -n "$K" ]; then timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" 2>&1 | tail -4; fi
for r in $(seq $RUNS); do
  timeout 300 python bench.py --no-cpu-baseline --no-max-context --no-e2e --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()}, d['clocks']['reasons'])"
done
if [ "$TK" != none ]; then timeout 300 python tools/trace_kernel.py --kernel $TK --cta-table > gpurun_out/trace_$TK.txt 2>&1; head -12 gpurun_out/trace_$TK.txt; fi
