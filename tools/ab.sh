#!/bin/bash
# A/B the in-tree library against scratch/base.so on the same box (alternating runs).
#   bash tools/ab.sh [rounds] [bench args...]
R=${1:-3}; shift
for i in $(seq 1 $R); do
  for lib in scratch/base.so paper_2510_04008_b200/librace_b200.so; do
    RACE_LIB_PATH=$PWD/$lib python bench.py --no-cpu-baseline --no-max-context --no-e2e "$@" 2>&1 | tail -1 > gpurun_out/ab.json
    python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print(sys.argv[1].split('/')[-1], round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()})" $lib
  done
done
