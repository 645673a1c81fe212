# ck8 with E in its own TMEM columns (issued one chunk ahead), dX over the EG~/P~ columns; no-stack build
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -q -p no:cacheprovider -x -k "fast_path or config1 or kside_rows or golden_bf16 or hyperparameters or small_n or batch_head or inplace or narrow or fast_groups or headline" 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --no-max-context --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])"; done
