# CUDA-core path: segment size sweep (fp32 causal / non-causal) + generic-path parity
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "config1 and f32 or table_groups or golden_fp32 or inplace" 2>&1 | tail -1
for t in 1184 1776 2072 4096; do
  for c in "" "--noncausal"; do
    RACE_SIMT_SEG_TARGET=$t timeout 300 python bench.py --dtype f32 $c --steps 10 --no-max-context --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t $c', round(d['value']/1e6,1), 'M tok/s', {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()})"
  done
done
