set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpt.py -q -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do timeout 600 python bench.py --no-max-context --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e6, d['e2e'])"; done
timeout 600 python - <<'PY'
import sys, torch, json
sys.path.insert(0, '.')
import bench
print(json.dumps(bench.gpt_train_step(torch.device('cuda', 0))))
PY
