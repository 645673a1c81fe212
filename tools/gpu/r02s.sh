set -x
mkdir -p gpurun_out
export RACE_PARITY_LOG=gpurun_out/r02s_parity.jsonl
rm -f $RACE_PARITY_LOG
timeout 1200 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "fast_groups or wide or table_groups or inplace or golden_bf16" 2>&1 | tail -3
timeout 600 python - <<'PY'
import sys, json, torch
sys.path.insert(0, '.')
import bench
bench.sketch_sweep(torch.device('cuda', 0), torch.bfloat16)  # warm
for r in bench.sketch_sweep(torch.device('cuda', 0), torch.bfloat16): print(r)
PY
