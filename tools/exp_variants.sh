#!/bin/bash
# Rebuild the library with each macro set and time the search kernel on the bench index; dev tool.
# Usage: bash tools/exp_variants.sh "<L list>" "-DX=1 -DY=2" "-DX=2" ...
LS=$1; shift
for v in "$@"; do
  touch paper_2601_07048_b200/csrc/search.cu
  JB_NVCC_EXTRA="$v" python -m paper_2601_07048_b200._build > /dev/null || { echo "build failed: $v"; continue; }
  for reg in ${JB_EXP_REGS:-0 1}; do
    JB_SEARCH_REG=$reg JB_EXP_HS=${JB_EXP_HS:-0} timeout 600 python tools/exp_search.py $LS 2>&1 | grep MQPS | sed "s/^/[$v reg=$reg] /"
  done
done
touch paper_2601_07048_b200/csrc/search.cu
