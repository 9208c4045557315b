#!/bin/bash
# Run on the GPU box via gpurun: bench line + ncu launch list + one ncu --set full of the search kernel.
# Usage: bash profiles/profile_round.sh <tag> [extra bench args]
set -x
TAG=${1:-r01}; shift
mkdir -p gpurun_out
timeout 900 python bench.py "$@" --out gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.log
tail -5 gpurun_out/bench_${TAG}.log
L=$(python -c "import json;print(json.load(open('gpurun_out/bench_${TAG}.json'))['config']['beam_width'])")
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py "$@" --beam $L --no-cpu --steps 3 --warmup 1 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
    -k regex:beam_search_kernel -c 1 -o gpurun_out/prof_search_${TAG} -f python bench.py "$@" --beam $L --no-cpu \
    --steps 1 --warmup 1 > gpurun_out/ncu_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_${TAG}.log
ls -la gpurun_out
