#!/bin/bash
# construction variants: 1M x 128 bulk build (3 reps) and one 100K batch into 3M x 96 (dev tool)
for v in "$@"; do
  touch paper_2601_07048_b200/csrc/build.cu
  JB_NVCC_EXTRA="$v" python -m paper_2601_07048_b200._build > /dev/null || { echo "build failed $v"; continue; }
  JB_EXP_REPS=3 timeout 600 python tools/exp_build_prof.py 2>&1 | grep "^build" | sed "s/; work.*//" | tail -2 | sed "s/^/[$v] /"
  JB_PROFILE=1 timeout 900 python tools/exp_stream_prof.py 3000000 1 2>&1 | grep -E "^\[jb\] batch \[3000000" | sed "s/^/[$v] /"
done
touch paper_2601_07048_b200/csrc/build.cu
