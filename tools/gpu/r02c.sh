# round-2 pass c: M=64 two-chain selftest, fixed k-rows test, eager vs graph, ncu of the headline and fp32 (SIMT) steps
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_tc_selftest.py tests/test_gpu_parity.py -k "selftest or m64 or kside_rows" -q -p no:cacheprovider 2>&1 | tail -5
timeout 300 python tools/eager_vs_graph.py 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_launches_causal.csv python tools/profile_step.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_aggregate2|k_causal_fwd8|k_bwd_causal|k_combine" -s 6 -c 6 -o gpurun_out/r02c_causal python tools/profile_step.py > gpurun_out/r02c_ncu_causal.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -s 7 -c 7 -o gpurun_out/r02c_f32_causal python tools/profile_step.py --dtype f32 > gpurun_out/r02c_ncu_f32.log 2>&1
ls -la gpurun_out
