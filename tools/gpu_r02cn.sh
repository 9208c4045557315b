#!/bin/bash
# bit-exact RaBitQ kernel at 12 resident blocks vs 8: C5 shard (m=4) and C2 (m=1, reference estimator)
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
for b in 8 12; do
  JB_RQ_BLOCKS=$b timeout 900 python bench.py --config c5 --beam 80 --estimator reference --no-cpu --steps 10 --warmup 3 --out gpurun_out/rq_c5_$b.json > gpurun_out/rq_c5_$b.log 2>&1
  python -c "import json;b=json.load(open('gpurun_out/rq_c5_$b.json'));print('c5 blocks $b', b['value'], b['kernel_ms']['search'], b['e2e']['value'])"
done
for b in 8 12; do
  JB_RQ_BLOCKS=$b timeout 900 python bench.py --beam 128 --estimator reference --no-cpu --steps 10 --warmup 3 --out gpurun_out/rq_c2_$b.json > gpurun_out/rq_c2_$b.log 2>&1
  python -c "import json;b=json.load(open('gpurun_out/rq_c2_$b.json'));print('c2 blocks $b', b['value'], b['kernel_ms']['search'])"
done
