#!/bin/bash
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_screen_gpu.py tests/test_build_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_ch.log 2>&1
tail -1 gpurun_out/pytest_ch.log
timeout 900 python tools/exp_build_ab.py "JB_SCREEN_MINB=8,JB_SCREEN_SROWS=16" "JB_SCREEN_MINB=14,JB_SCREEN_SROWS=8" 2>&1 | tail -2
