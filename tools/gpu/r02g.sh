# SIMT tile-size A/B (fp32 inputs run on the generic path): parity of each variant + fp32 bench lines
set -x
mkdir -p gpurun_out
for lib in paper_2510_04008_b200/librace_b200.so scratch/t16.so scratch/t64.so; do
  echo "== $lib"
  RACE_LIB_PATH=$PWD/$lib timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "config1 and f32 or table_groups or golden_fp32" 2>&1 | tail -1
  for c in "" "--noncausal"; do
    RACE_LIB_PATH=$PWD/$lib timeout 300 python bench.py --dtype f32 $c --steps 10 --no-max-context --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']/1e6,1), 'M tok/s', {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()})"
  done
done
