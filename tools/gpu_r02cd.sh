#!/bin/bash
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 300 python tools/exp_py_overhead.py 2>&1 | tail -6
JB_PIPE_PROFILE=1 timeout 300 python tools/exp_e2e_first.py 0 2>&1 | grep -E "jb pipeline" | tail -4
