#!/bin/bash
# full search_knn_batch step (two lanes: bind + search + rerank) over compile-time variants (dev tool)
for v in "$@"; do
  touch paper_2601_07048_b200/csrc/search.cu
  JB_NVCC_EXTRA="$v" python -m paper_2601_07048_b200._build > /dev/null || { echo "build failed $v"; continue; }
  timeout 600 python tools/exp_host_chunks.py 0 0 2>&1 | grep -E "chunk|device API" | sed "s/^/[$v] /"
done
touch paper_2601_07048_b200/csrc/search.cu
python -m paper_2601_07048_b200._build > /dev/null
