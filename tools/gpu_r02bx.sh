#!/bin/bash
# screen with a smaller stage (more warps/SM): tests, phase-1 search A/B over stage rows, build A/B
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_screen_gpu.py tests/test_search_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_bx.log 2>&1
tail -2 gpurun_out/pytest_bx.log
for r in 8 16 32; do JB_SCREEN_SROWS=$r timeout 600 python tools/exp_screen.py 2>&1 | tail -2 | sed "s/^/srows=$r /"; done
timeout 900 python tools/exp_build_ab.py "JB_SCREEN=0" "JB_SCREEN=1,JB_SCREEN_SROWS=16" "JB_SCREEN=1,JB_SCREEN_SROWS=8" 2>&1 | tail -3
