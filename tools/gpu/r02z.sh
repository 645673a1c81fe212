set -x
bash tools/gpu/r02s.sh
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-max-context --no-e2e --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()}, d['clocks']['reasons'])"; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z_grouped_p2l4.csv python tools/profile_grouped.py --P 2 --L 4 > /dev/null 2>&1
