#!/bin/bash
# ncu --set full of the search kernel, register beam (reg=1) vs smem beam (reg=0); dev tool.
mkdir -p gpurun_out
L=${1:-128}; EST=${2:-popcount}; TAG=${3:-ab}
for reg in 1 0; do
  JB_SEARCH_REG=$reg timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" \
    -k regex:beam_search -c 1 -o gpurun_out/prof_${TAG}_reg$reg -f python tools/exp_prof_search.py $L $EST > gpurun_out/ncu_${TAG}_reg$reg.log 2>&1
  tail -2 gpurun_out/ncu_${TAG}_reg$reg.log
done
