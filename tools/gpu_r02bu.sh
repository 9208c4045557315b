#!/bin/bash
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 600 python tools/exp_screen.py 2>&1 | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:beam_search_kernel --launch-skip 60 -c 4 --csv python tools/exp_screen.py 2>/dev/null | grep -E "dram__bytes_read|gpu__time|inst_executed|hit_rate" | awk -F'","' '{print $(NF-2), $(NF-1), $(NF)}'
