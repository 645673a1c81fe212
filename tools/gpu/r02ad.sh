set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpt.py tests/test_sharded_gpu.py -q -p no:cacheprovider -x -k "narrow or gpt or d64 or fast_path or config1 or batch_head or inplace or fast_groups or golden_bf16 or sharding or kside_rows or misaligned" 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline --no-max-context --no-e2e --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()})"
timeout 600 python - <<'PY'
import sys, torch, json
sys.path.insert(0, '.')
import bench
print(json.dumps(bench.gpt_train_step(torch.device('cuda', 0))))
PY
