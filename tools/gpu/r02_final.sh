# round-2 measurement set: bench lines (headline with max context / sweeps / GPT, non-causal, fp32,
# reference arm), ncu launch list of bench.py itself, ncu --set full of the causal / non-causal steps
# and of the fp32 (CUDA-core) causal step, GPT-step kernel profile
set -x
mkdir -p gpurun_out
R=${1:-r02n}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python bench.py > gpurun_out/${R}_bench.log 2>&1; tail -1 gpurun_out/${R}_bench.log > gpurun_out/${R}_bench_causal.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${R}_ref.log 2>&1; tail -1 gpurun_out/${R}_ref.log > gpurun_out/${R}_bench_reference_arm.json
timeout 600 python bench.py --noncausal --no-max-context > gpurun_out/${R}_nc.log 2>&1; tail -1 gpurun_out/${R}_nc.log > gpurun_out/${R}_bench_noncausal.json
timeout 600 python bench.py --dtype f32 --no-max-context --no-e2e --steps 20 > gpurun_out/${R}_f32c.log 2>&1; tail -1 gpurun_out/${R}_f32c.log > gpurun_out/${R}_bench_f32_causal.json
timeout 600 python bench.py --dtype f32 --noncausal --no-max-context --no-e2e --steps 20 > gpurun_out/${R}_f32nc.log 2>&1; tail -1 gpurun_out/${R}_f32nc.log > gpurun_out/${R}_bench_f32_noncausal.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-max-context --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_aggregate2|k_causal_fwd8|k_bwd_causal|k_combine" -s 6 -c 6 -o gpurun_out/${R}_causal python tools/profile_step.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_aggregate2|k_readout8|k_bwd_q8|k_bwd_k8|k_combine" -s 6 -c 6 -o gpurun_out/${R}_noncausal python tools/profile_step.py --noncausal > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -s 7 -c 7 -o gpurun_out/${R}_f32_causal python tools/profile_step.py --dtype f32 > /dev/null 2>&1
timeout 600 python tools/profile_gpt.py > gpurun_out/${R}_gpt_profile.txt 2>&1
ls -la gpurun_out | tail -20
