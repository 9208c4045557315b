#!/bin/bash
# column-sum loaders batched + lazy host graph slab: parity tests, medoid timing, 1M build profile
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_rabitq_props.py tests/test_search_gpu.py tests/test_build_gpu.py tests/test_boundary_gpu.py tests/test_persistence.py -q -x -p no:cacheprovider > gpurun_out/pytest_bm.log 2>&1
tail -3 gpurun_out/pytest_bm.log
timeout 300 python tools/exp_medoid.py 2>&1 | tail -2
timeout 300 python tools/exp_medoid.py 12500000 96 2>&1 | tail -1
JB_EXP_PROFILE=1 JB_EXP_REPS=2 timeout 600 python tools/exp_build_prof.py > gpurun_out/bm_prof.log 2>&1
grep -E "medoid|^build|wall \[0, 33\)" gpurun_out/bm_prof.log
