# fast groups: parity (new tests + golden + groups) and the sketch sweep
set -x
mkdir -p gpurun_out
export RACE_PARITY_LOG=gpurun_out/r02h_parity.jsonl
rm -f $RACE_PARITY_LOG
timeout 1200 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "fast_groups or wide or table_groups or golden or fast_path_hyper" 2>&1 | tail -8
timeout 600 python - <<'PY'
import sys, json, torch
sys.path.insert(0, '.')
import bench
print(json.dumps(bench.sketch_sweep(torch.device('cuda', 0), torch.bfloat16)))
PY
