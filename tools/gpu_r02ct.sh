#!/bin/bash
# verification after the screen: full GPU suite, smoke, profile round (C2), C5 shard bench, configs c3 c4 c1
set -x
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > gpurun_out/build_ct.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_ct.log 2>&1
tail -3 gpurun_out/pytest_gpu_ct.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_ct.log 2>&1
tail -2 gpurun_out/smoke_ct.log
bash profiles/profile_round.sh r02ct --steps 10 --warmup 3
timeout 1200 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu --out gpurun_out/bench_r02ct_c5.json > gpurun_out/bench_r02ct_c5.log 2>&1
tail -2 gpurun_out/bench_r02ct_c5.log
bash tools/run_configs.sh c4
