#!/bin/bash
# screen policy with smem next-hop staging beyond 3 x L2: tests, C5 shard bench, C4 config, 1M build
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_screen_gpu.py tests/test_build_gpu.py tests/test_closure_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_cp.log 2>&1
tail -1 gpurun_out/pytest_cp.log
timeout 1200 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu --out gpurun_out/bench_r02cp_c5.json > gpurun_out/bench_r02cp_c5.log 2>&1
python -c "import json;b=json.load(open('gpurun_out/bench_r02cp_c5.json'));sk=b['build']['search_kernel_roofline'];print('c5', b['value'], b['build']['inserts_per_s'], sk['kernel_ms'], (sk.get('screened') or {}).get('kernel_ms'))"
bash tools/run_configs.sh c4
timeout 900 python tools/exp_build_ab.py "JB_SCREEN_FORCE=1" 2>&1 | tail -1
