set -x
mkdir -p gpurun_out
export RACE_PARITY_LOG=gpurun_out/r02d_probe.jsonl
timeout 300 python -m pytest tests/test_tc_selftest.py -q -p no:cacheprovider 2>&1 | tail -5
ls gpurun_out
