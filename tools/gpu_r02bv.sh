#!/bin/bash
# screen + chain-split A1: tests, phase-1 search A/B, 1M build A/B
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_screen_gpu.py tests/test_search_gpu.py tests/test_build_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_bv.log 2>&1
tail -3 gpurun_out/pytest_bv.log
timeout 600 python tools/exp_screen.py 2>&1 | tail -2
timeout 900 python tools/exp_build_ab.py "JB_SCREEN=0" "JB_SCREEN=1" 2>&1 | tail -2
