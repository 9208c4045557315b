#!/bin/bash
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python tools/exp_build_ab.py "JB_CLOSED_PASS=0" "JB_CLOSED_PASS=1,JB_CLOSED_EXTRA=6" "JB_CLOSED_PASS=1,JB_CLOSED_EXTRA=8" "JB_CLOSED_PASS=1,JB_CLOSED_EXTRA=12" "JB_CLOSED_PASS=1,JB_CLOSED_EXTRA=16" 2>&1 | tail -5
