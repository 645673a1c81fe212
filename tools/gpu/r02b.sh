# round-2: full GPU suite with the parity log (no -x: report every failure)
set -x
mkdir -p gpurun_out
export RACE_PARITY_LOG=gpurun_out/r02b_parity.jsonl
rm -f $RACE_PARITY_LOG
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > gpurun_out/r02b_gputest.log 2>&1; tail -40 gpurun_out/r02b_gputest.log
