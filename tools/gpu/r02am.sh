set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "causal and (fast or headline)" 2>&1 | tail -2
for r in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --no-max-context --no-e2e --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()}, d['clocks']['reasons'])"
done
timeout 300 python tools/trace_kernel.py --kernel bk --events 30 > gpurun_out/trace_bk30.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02am_grouped_p4l4.csv python tools/profile_grouped.py --P 4 --L 4 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/r02am_grouped_p4l4.csv 2>&1 | head -24
