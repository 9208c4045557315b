#!/bin/bash
# ncu of one owner-merge launch (3M-row stream, batch ~25), flat vs split prune (dev tool)
for v in "" "-DJB_OWNER_SPLIT"; do
  tag=${v:+split}; tag=${tag:-flat}
  touch paper_2601_07048_b200/csrc/build.cu
  JB_NVCC_EXTRA="$v" python -m paper_2601_07048_b200._build > /dev/null || { echo "build failed $v"; continue; }
  ncu --set full --import-source on --clock-control none -k regex:owner_merge_kernel --launch-skip 25 -c 1 \
    -o gpurun_out/prof_owner_$tag python tools/exp_stream_prof.py 3000000 1 > gpurun_out/ncu_owner_$tag.log 2>&1
done
touch paper_2601_07048_b200/csrc/build.cu
python -m paper_2601_07048_b200._build > /dev/null
