#!/bin/bash
# screen policy (records <= 2 x L2 or D >= 256): C5 shard bench, c4 config, tests
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_screen_gpu.py tests/test_build_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_ca.log 2>&1
tail -1 gpurun_out/pytest_ca.log
timeout 1200 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu --out gpurun_out/bench_r02ca_c5.json > gpurun_out/bench_r02ca_c5.log 2>&1
python -c "import json;b=json.load(open('gpurun_out/bench_r02ca_c5.json'));print('c5', b['value'], b['e2e']['value'], b['build']['inserts_per_s'], b['build']['search_kernel_roofline']['kernel_ms'])"
bash tools/run_configs.sh c4
