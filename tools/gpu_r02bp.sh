#!/bin/bash
# closed-row owner pass (MODE 3, staged, fewer rows): parity + 1M build A/B over the staging size
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_build_gpu.py tests/test_closure_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_bp.log 2>&1
tail -2 gpurun_out/pytest_bp.log
for v in "1 2" "1 4" "1 8" "0 4"; do
  set -- $v
  JB_CLOSED_PASS=$1 JB_CLOSED_EXTRA=$2 JB_EXP_REPS=2 timeout 600 python tools/exp_build_prof.py 2>&1 | grep "^build" | tail -1 | cut -c1-60 | sed "s/^/closed_pass=$1 extra=$2 /"
done
