#!/bin/bash
# A/B the search kernels (register beam vs smem beam) on the bench index; dev tool.
mkdir -p gpurun_out
for reg in 1 0; do
  JB_SEARCH_REG=$reg JB_EXP_HS="${JB_EXP_HS:-0}" timeout 600 python tools/exp_search.py "$@" 2>&1 | sed "s/^/reg=$reg /"
done
