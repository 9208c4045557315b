#!/bin/bash
# ncu --set full of the phase-1 search kernel unscreened and screened (1M x 128, 100K queries, L=64)
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
JB_EXP_NCU=1 timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:beam_search_kernel \
   -o gpurun_out/prof_p1_screen -f python tools/exp_screen.py > gpurun_out/ncu_p1.log 2>&1
tail -2 gpurun_out/ncu_p1.log
python profiles/summarize_ncu.py gpurun_out/prof_p1_screen.ncu-rep gpurun_out/p1_screen_summary.txt > /dev/null 2>&1
grep -E "## kernel|gpu__time|dram__bytes_read|issue_active|warps_active|inst_executed.sum|registers|shared_mem_per_block|occupancy_limit" gpurun_out/p1_screen_summary.txt
sed -n '/warp stall/,/^$/p' gpurun_out/p1_screen_summary.txt | head -30
