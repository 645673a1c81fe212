set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "fast_groups or wide or table_groups or golden or inplace" 2>&1 | tail -3
timeout 600 python - <<'PY'
import sys, json, torch
sys.path.insert(0, '.')
import bench
bench.sketch_sweep(torch.device('cuda', 0), torch.bfloat16)  # warm
for r in bench.sketch_sweep(torch.device('cuda', 0), torch.bfloat16): print(r)
PY
