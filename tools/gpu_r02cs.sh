#!/bin/bash
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python tools/exp_build_ab.py "JB_SCREEN_NEXT=0" "JB_SCREEN_FORCE=1" "JB_SCREEN_FORCE=0" 2>&1 | tail -3
for i in 1 2; do
timeout 900 python bench.py --beam 128 --no-cpu --steps 5 --warmup 3 --out gpurun_out/bcheck_$i.json > gpurun_out/bcheck_$i.log 2>&1
python -c "import json;b=json.load(open('gpurun_out/bcheck_$i.json'));print('bench build', b['build']['inserts_per_s'], b['build']['build_s'])"
done
