# shared-memory provenance (LDS/STS instead of generic LD/ST) + printf-free waits: parity + timing
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -q -p no:cacheprovider -x -k "fast_path or config1 or kside_rows or golden_bf16 or hyperparameters or small_n or batch_head or inplace or narrow" 2>&1 | tail -3
timeout 600 python bench.py --no-max-context --no-cpu-baseline > gpurun_out/r02e_bench.log 2>&1; tail -1 gpurun_out/r02e_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['e2e']['value'])"
timeout 600 python bench.py --noncausal --no-max-context --no-cpu-baseline --no-e2e > gpurun_out/r02e_bench_nc.log 2>&1; tail -1 gpurun_out/r02e_bench_nc.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])"
