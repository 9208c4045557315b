#!/bin/bash
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
for pf in 0 1; do JB_SCREEN_PF=$pf timeout 600 python tools/exp_screen.py 2>&1 | tail -1 | sed "s/^/pf=$pf /"; done
timeout 900 python tools/exp_build_ab.py "JB_SCREEN_PF=0" "JB_SCREEN_PF=1" 2>&1 | tail -2
