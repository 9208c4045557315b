#!/bin/bash
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
JB_EXP_NCU=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:beam_search_kernel --csv python tools/exp_screen.py 2>/dev/null | grep -E "beam_search" | awk -F'","' '{print $(NF-2), $(NF-1), $(NF)}'
