set -x
mkdir -p gpurun_out
for r in 1 2 3; do
for lib in paper_2510_04008_b200/librace_b200.so scratch/ck8e.so; do
  RACE_LIB_PATH=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --no-max-context --no-e2e --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()}, d['clocks']['reasons'])"
done; done
RACE_LIB_PATH=$PWD/scratch/ck8e.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -q -p no:cacheprovider -x -k "fast_path_backward and causal or headline_config_all_heads_vs_oracle and causal or hyperparameters and _c" 2>&1 | tail -2
bash tools/gpu/r02_ncu.sh r02o
