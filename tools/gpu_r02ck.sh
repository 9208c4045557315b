#!/bin/bash
# next-hop screen-record prefetch: none / prefetch.global.L2 / cp.async.bulk.prefetch.L2 at 1M x 128 and 6M x 96
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
for pf in 0 1 2; do JB_SCREEN_PF=$pf timeout 600 python tools/exp_screen.py 2>&1 | tail -1 | sed "s/^/1M pf=$pf /"; done
for pf in 1 2; do JB_SCREEN_PF=$pf JB_EXP_N=6000000 JB_EXP_D=96 timeout 900 python tools/exp_screen.py 2>&1 | tail -2 | sed "s/^/6M pf=$pf /"; done
