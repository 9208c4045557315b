#!/bin/bash
# re-entry verification of HEAD: full GPU suite, smoke, profile round (bench + launch list + ncu full)
set -x
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > gpurun_out/build_bh.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_bh.log 2>&1
tail -3 gpurun_out/pytest_gpu_bh.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_bh.log 2>&1
tail -2 gpurun_out/smoke_bh.log
bash profiles/profile_round.sh r02bh --steps 10 --warmup 3
