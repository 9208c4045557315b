#!/bin/bash
# screen at HBM-resident scale (12.5M x 96 and 3M x 96) with the 8-row / 14-block kernel
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
JB_EXP_N=6000000 JB_EXP_D=96 timeout 900 python tools/exp_screen.py 2>&1 | tail -2 | sed "s/^/6M x 96 /"
JB_EXP_N=4500000 JB_EXP_D=96 timeout 900 python tools/exp_screen.py 2>&1 | tail -2 | sed "s/^/4.5M x 96 /"
