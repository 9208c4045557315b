#!/bin/bash
# column-sum kernel rewrite: parity tests + 1M build phase profile
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_rabitq_props.py tests/test_search_gpu.py tests/test_build_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_bk.log 2>&1
tail -3 gpurun_out/pytest_bk.log
JB_EXP_PROFILE=1 JB_EXP_REPS=2 timeout 600 python tools/exp_build_prof.py > gpurun_out/bk_prof.log 2>&1
grep -E "medoid|^build" gpurun_out/bk_prof.log
