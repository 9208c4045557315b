#!/bin/bash
# int8 screen of the exact search: tests + 1M build A/B (identical graphs, time)
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_screen_gpu.py tests/test_abi.py -q -x -p no:cacheprovider > gpurun_out/pytest_bt.log 2>&1
tail -15 gpurun_out/pytest_bt.log
timeout 900 python tools/exp_build_ab.py "JB_SCREEN=0" "JB_SCREEN=1" 2>&1 | tail -3
JB_PROFILE=1 timeout 300 python tools/exp_build_prof.py 2>&1 | grep -E "batch \[835135" 
JB_SCREEN=0 JB_PROFILE=1 timeout 300 python tools/exp_build_prof.py 2>&1 | grep -E "batch \[835135"
