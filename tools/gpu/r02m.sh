# same-box A/B: head (groups, runtime-indexed) / nock8 (compile-time idx) / current (HB template param)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -q -p no:cacheprovider -x -k "fast_path_backward or config1 or fast_groups or hyperparameters" 2>&1 | tail -2
for r in 1 2; do
for lib in scratch/nock8.so paper_2510_04008_b200/librace_b200.so; do
  RACE_LIB_PATH=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --no-max-context --no-e2e --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()})"
done; done
