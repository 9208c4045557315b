#!/bin/bash
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_screen_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_cq.log 2>&1
tail -1 gpurun_out/pytest_cq.log
