#!/bin/bash
# construction kernels: staging budget variants, 1M x 128 bulk build (dev tool)
for v in "$@"; do
  touch paper_2601_07048_b200/csrc/build.cu
  JB_NVCC_EXTRA="$v" python -m paper_2601_07048_b200._build > /dev/null || { echo "build failed $v"; continue; }
  for rep in 1; do
    JB_EXP_REPS=3 timeout 600 python tools/exp_build_prof.py 2>&1 | grep "^build" | sed "s/; work.*//" | sed "s/^/[$v] /"
  done
done
touch paper_2601_07048_b200/csrc/build.cu
