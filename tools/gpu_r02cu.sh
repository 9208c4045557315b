#!/bin/bash
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 600 python -m pytest tests/test_rabitq_props.py -q -p no:cacheprovider -k "row_sq_norms or column_mean" > gpurun_out/pytest_cu.log 2>&1
tail -3 gpurun_out/pytest_cu.log
