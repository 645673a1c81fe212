set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dx_from_dproj -s 2 -c 1 -o gpurun_out/r02ah_dx python tools/profile_grouped.py --P 2 --L 4 > gpurun_out/r02ah_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_group_fwd_acc -s 2 -c 1 -o gpurun_out/r02ah_facc python tools/profile_grouped.py --P 2 --L 4 >> gpurun_out/r02ah_ncu.log 2>&1
ls -la gpurun_out/
