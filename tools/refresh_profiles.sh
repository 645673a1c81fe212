set -x
python bench.py > gpurun_out/r01f_bench.log 2>&1; tail -1 gpurun_out/r01f_bench.log > gpurun_out/r01f_bench.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01f_ref.log 2>&1; tail -1 gpurun_out/r01f_ref.log > gpurun_out/r01f_ref.json
python bench.py --noncausal --no-max-context --no-cpu-baseline > gpurun_out/r01f_nc.log 2>&1; tail -1 gpurun_out/r01f_nc.log > gpurun_out/r01f_bench_noncausal.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01f_launches.csv python tools/profile_step.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_aggregate2|k_causal_fwd8|k_bwd_causal|k_combine" -s 6 -c 6 -o gpurun_out/prof_r01f_causal python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
