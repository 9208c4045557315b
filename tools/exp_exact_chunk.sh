#!/bin/bash
# exact-source search staging chunk variants: 1M x 128 bulk build phase-1 search + C1 search (dev tool)
for v in "$@"; do
  touch paper_2601_07048_b200/csrc/search.cu
  JB_NVCC_EXTRA="$v" python -m paper_2601_07048_b200._build > /dev/null || { echo "build failed $v"; continue; }
  JB_EXP_REPS=1 JB_EXP_PROFILE=1 timeout 600 python tools/exp_build_prof.py 2>&1 | grep -E "batch \[(835135|935135)" | sed "s/^/[$v] /"
  timeout 600 python bench_configs.py c1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v] c1', [(p['L'], p['qps_device']) for p in d['sweep']])"
done
touch paper_2601_07048_b200/csrc/search.cu
