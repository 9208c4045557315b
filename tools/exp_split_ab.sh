#!/bin/bash
# split vs flat staged prune: per-phase build times at 1M and 3M rows, 96-d (dev tool)
for v in "-DJB_NO_SPLIT" ""; do
  touch paper_2601_07048_b200/csrc/build.cu
  JB_NVCC_EXTRA="$v" python -m paper_2601_07048_b200._build > /dev/null || { echo "build failed $v"; continue; }
  JB_PROFILE=1 timeout 600 python tools/exp_stream_prof.py 3000000 1 2>&1 \
    | grep -E "^\[jb\] batch \[(535135|900000|2900000|3000000)" | sed "s/^/[$v] /"
done
touch paper_2601_07048_b200/csrc/build.cu
python -m paper_2601_07048_b200._build > /dev/null
