#!/bin/bash
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
for v in "8 16" "14 16" "14 8" "8 8"; do set -- $v
  JB_SCREEN_MINB=$1 JB_SCREEN_SROWS=$2 timeout 600 python tools/exp_screen.py 2>&1 | tail -1 | sed "s/^/minb=$1 srows=$2 /"
done
