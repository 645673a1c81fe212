set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "group or wide or golden or grouped or P11 or sketch" 2>&1 | tail -3
timeout 600 python tools/sketch_sweep.py
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02ai_grouped_p2l4.csv python tools/profile_grouped.py --P 2 --L 4 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/r02ai_grouped_p2l4.csv 2>&1 | head -20
