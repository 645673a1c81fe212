set -x
for r in 1 2 3; do
for lib in scratch/base.so paper_2510_04008_b200/librace_b200.so; do
  RACE_LIB_PATH=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --no-max-context --no-e2e --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()}, d['clocks']['reasons'])"
done; done
timeout 600 python -c "
import torch, bench
print('gpt', bench.gpt_train_step(torch.device('cuda', 0)))
"
