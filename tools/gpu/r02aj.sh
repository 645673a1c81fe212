set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "group or wide or grouped or P11" 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02aj_grouped_p2l4.csv python tools/profile_grouped.py --P 2 --L 4 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/r02aj_grouped_p2l4.csv 2>&1 | grep -E "dx_from|group_"
