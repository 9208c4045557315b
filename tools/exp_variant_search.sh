#!/bin/bash
# search kernel A/B over compile-time variants: bash tools/exp_variant_search.sh "<flags A>" "<flags B>" ... (dev tool)
for v in "$@"; do
  touch paper_2601_07048_b200/csrc/search.cu
  JB_NVCC_EXTRA="$v" python -m paper_2601_07048_b200._build > /dev/null || { echo "build failed $v"; continue; }
  JB_EXP_HS=0 timeout 600 python tools/exp_search.py 64 128 2>&1 | grep MQPS | sed "s/^/[$v] /"
done
touch paper_2601_07048_b200/csrc/search.cu
python -m paper_2601_07048_b200._build > /dev/null
