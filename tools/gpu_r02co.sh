#!/bin/bash
# next-hop screen records staged in smem (JB_SCREEN_NEXT=1): parity, then phase-1 timing at 1M x 128, 6M / 12.5M x 96
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
JB_SCREEN_NEXT=1 timeout 900 python -m pytest tests/test_screen_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_co.log 2>&1
tail -1 gpurun_out/pytest_co.log
for nx in 0 1; do JB_SCREEN_NEXT=$nx timeout 600 python tools/exp_screen.py 2>&1 | tail -1 | sed "s/^/1M next=$nx /"; done
for nx in 0 1; do JB_SCREEN_NEXT=$nx JB_EXP_N=6000000 JB_EXP_D=96 timeout 900 python tools/exp_screen.py 2>&1 | tail -2 | sed "s/^/6M next=$nx /"; done
JB_SCREEN_NEXT=1 JB_EXP_N=12500000 JB_EXP_D=96 timeout 1200 python tools/exp_screen.py 2>&1 | tail -2 | sed "s/^/12.5M next=1 /"
