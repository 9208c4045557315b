#!/bin/bash
# closed-row owner pass (MODE 3): parity + 1M build A/B
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_build_gpu.py tests/test_closure_gpu.py tests/test_donor_tc_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_bo.log 2>&1
tail -3 gpurun_out/pytest_bo.log
for v in 1 0; do
  JB_CLOSED_PASS=$v JB_EXP_REPS=2 timeout 600 python tools/exp_build_prof.py 2>&1 | grep "^build" | sed "s/^/closed_pass=$v /"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"owner_merge" --csv \
   python tools/exp_build_prof.py 2>/dev/null | grep gpu__time | awk -F'","' '{print $5, $(NF)}' | tail -8
