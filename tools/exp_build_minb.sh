#!/bin/bash
# phase-1 search occupancy (JB_OTHER_MINB) vs bulk-build phase times, 1M x 128 (dev tool)
for v in "$@"; do
  touch paper_2601_07048_b200/csrc/search.cu
  JB_NVCC_EXTRA="$v" python -m paper_2601_07048_b200._build > /dev/null || { echo "build failed $v"; continue; }
  JB_EXP_PROFILE=1 JB_EXP_REPS=2 timeout 600 python tools/exp_build_prof.py 2>&1 | python -c "
import re, sys
tot = {}; lines = sys.stdin.read().splitlines()
rows = [l for l in lines if l.startswith('[jb] batch [')]
for l in rows[len(rows) // 2:]:
    for k, val in re.findall(r'(\w+) ([\d.]+)ms', l): tot[k] = tot.get(k, 0) + float(val)
print('[$v]', {k: round(val, 1) for k, val in tot.items()}, [l[:40] for l in lines if l.startswith('build')][-1:])"
done
touch paper_2601_07048_b200/csrc/search.cu
python -m paper_2601_07048_b200._build > /dev/null
