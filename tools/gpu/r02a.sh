# round-2 first GPU pass: full GPU suite (with parity log), bench, reference arm, 2-rank bench on one GPU
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
mkdir -p gpurun_out
export RACE_PARITY_LOG=gpurun_out/r02a_parity.jsonl
rm -f $RACE_PARITY_LOG
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02a_gputest.log 2>&1; tail -5 gpurun_out/r02a_gputest.log
timeout 900 python bench.py > gpurun_out/r02a_bench.log 2>&1; tail -1 gpurun_out/r02a_bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02a_ref.log 2>&1; tail -1 gpurun_out/r02a_ref.log
RACE_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --sharded-64m-total 8388608 > gpurun_out/r02a_bench2.log 2>&1; tail -3 gpurun_out/r02a_bench2.log
