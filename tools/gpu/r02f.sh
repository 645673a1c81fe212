# ncu --set full of the causal step after the LDS fix (source-level stall attribution)
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_aggregate2|k_causal_fwd8|k_bwd_causal|k_combine" -s 6 -c 6 -o gpurun_out/r02f_causal python tools/profile_step.py > gpurun_out/r02f_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_aggregate2|k_readout8|k_bwd_q8|k_bwd_k8|k_combine" -s 6 -c 6 -o gpurun_out/r02f_noncausal python tools/profile_step.py --noncausal > gpurun_out/r02f_ncu_nc.log 2>&1
ls -la gpurun_out | tail -3
