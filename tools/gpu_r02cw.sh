#!/bin/bash
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python tools/exp_build_ab.py "JB_P2S_EXTRA=16" "JB_P2S_EXTRA=4" "JB_P2S_EXTRA=8" "JB_P2S_EXTRA=32" 2>&1 | tail -4
