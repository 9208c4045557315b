#!/bin/bash
# int8-screened phase-2 prune: tests + 1M build A/B (+ 12.5M-shaped stream check via c4 later)
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_screen_gpu.py tests/test_build_gpu.py tests/test_closure_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_cb.log 2>&1
tail -3 gpurun_out/pytest_cb.log
timeout 900 python tools/exp_build_ab.py "JB_P2_SCREEN=0" "JB_P2_SCREEN=1" 2>&1 | tail -2
JB_EXP_PROFILE=1 timeout 300 python tools/exp_build_prof.py 2>&1 | grep -E "batch \[835135"
JB_P2_SCREEN=0 JB_EXP_PROFILE=1 timeout 300 python tools/exp_build_prof.py 2>&1 | grep -E "batch \[835135"
