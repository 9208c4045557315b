#!/bin/bash
# phase-3 owner merge staging variants at 3M x 96 (dev tool)
for v in "$@"; do
  touch paper_2601_07048_b200/csrc/build.cu
  JB_NVCC_EXTRA="$v" python -m paper_2601_07048_b200._build > /dev/null || { echo "build failed $v"; continue; }
  JB_PROFILE=1 timeout 900 python tools/exp_stream_prof.py 3000000 1 2>&1 | grep -E "^\[jb\] batch \[3000000" | sed "s/^/[$v] /"
done
touch paper_2601_07048_b200/csrc/build.cu
