# ncu --set full of the causal and non-causal bf16 steps (tcgen05 path)
set -x
mkdir -p gpurun_out
R=${1:-r02n}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_aggregate2|k_causal_fwd8|k_bwd_causal|k_combine" -s 6 -c 6 -o gpurun_out/${R}_causal python tools/profile_step.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_aggregate2|k_readout8|k_bwd_q8|k_bwd_k8|k_combine" -s 6 -c 6 -o gpurun_out/${R}_noncausal python tools/profile_step.py --noncausal > /dev/null 2>&1
du -sh gpurun_out
