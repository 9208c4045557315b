#!/bin/bash
# construction with / without the high-D dot-matrix kernels, default and bench params (dev tool)
for v in "-DJB_NO_MATRIX" ""; do
  touch paper_2601_07048_b200/csrc/build.cu
  JB_NVCC_EXTRA="$v" python -m paper_2601_07048_b200._build > /dev/null || { echo "build failed $v"; continue; }
  timeout 900 python tools/exp_build_r64.py 2>&1 | sed "s/^/[$v] /"
  timeout 900 python tools/exp_build_prof.py 300000 960 2>&1 | grep "^build" | cut -c1-50 | sed "s/^/[$v] /"
done
touch paper_2601_07048_b200/csrc/build.cu
python -m paper_2601_07048_b200._build > /dev/null
