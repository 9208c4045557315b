#!/bin/bash
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 300 python tools/exp_medoid.py 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"column_sum|medoid|row_sq" --csv python tools/exp_medoid.py 2>/dev/null | grep -E "gpu__time" | awk -F'","' '{print $5, $(NF)}' | head -20
