set -x
mkdir -p gpurun_out
export RACE_PARITY_LOG=gpurun_out/r02j_parity.jsonl
rm -f $RACE_PARITY_LOG
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02j_gputest.log 2>&1; tail -4 gpurun_out/r02j_gputest.log
timeout 600 python - <<'PY'
import sys, json, torch
sys.path.insert(0, '.')
import bench
bench.sketch_sweep(torch.device('cuda', 0), torch.bfloat16)  # warm
for r in bench.sketch_sweep(torch.device('cuda', 0), torch.bfloat16): print(r)
PY
