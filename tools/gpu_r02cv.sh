#!/bin/bash
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_cv.log 2>&1
tail -1 gpurun_out/pytest_gpu_cv.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --out gpurun_out/bench_cv.json > gpurun_out/bench_cv.log 2>&1
python -c "import json;b=json.load(open('gpurun_out/bench_cv.json'));print(b['value'], b['e2e']['value'], b['build']['inserts_per_s'], b['gpu_launches'])"
