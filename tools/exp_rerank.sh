#!/bin/bash
# rerank kernel variants (warps per block x staged rows) on the bench workload; dev tool
for v in "-DJB_RR_WARPS=4 -DJB_RR_ROWS=8" "-DJB_RR_WARPS=2 -DJB_RR_ROWS=8" "-DJB_RR_WARPS=1 -DJB_RR_ROWS=8" "-DJB_RR_WARPS=8 -DJB_RR_ROWS=8"; do
  touch paper_2601_07048_b200/csrc/search.cu
  JB_NVCC_EXTRA="$v" python -m paper_2601_07048_b200._build > /dev/null
  timeout 600 python bench.py --no-cpu --steps 5 --warmup 3 --out gpurun_out/rr.json 2>/dev/null > /dev/null
  python -c "import json; d=json.load(open('gpurun_out/rr.json')); print('$v', d['kernel_ms']['rerank'], d['value'])"
done
touch paper_2601_07048_b200/csrc/search.cu
