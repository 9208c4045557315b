#!/bin/bash
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 600 python tools/exp_e2e_first.py 0 500 1000 1500 2500 2>&1 | tail -7
