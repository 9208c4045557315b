#!/bin/bash
# 16-bit tagged visited table A/B: search parity tests, C2 (both estimators) and C5 shard
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > gpurun_out/build_bi.log 2>&1
timeout 900 python -m pytest tests/test_search_gpu.py tests/test_build_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_bi.log 2>&1
tail -2 gpurun_out/pytest_bi.log
for t in 0 1; do
  JB_TAG16=$t timeout 600 python bench.py --beam 128 --no-cpu --steps 10 --warmup 3 --out gpurun_out/bi_c2_t$t.json > gpurun_out/bi_c2_t$t.log 2>&1
  grep -E "\] \[(reference|popcount)\] L=" gpurun_out/bi_c2_t$t.log | sed "s/^/tag16=$t /"
done
JB_TAG16=1 timeout 600 python bench.py --beam 128 --no-cpu --steps 10 --warmup 3 --hash-slots 1024 --out gpurun_out/bi_c2_h1024.json > gpurun_out/bi_c2_h1024.log 2>&1
grep -E "\] \[(reference|popcount)\] L=" gpurun_out/bi_c2_h1024.log | sed "s/^/tag16 h1024 /"
for v in "0 0" "1 1024" "0 1024"; do
  set -- $v
  JB_TAG16=$1 timeout 900 python bench.py --config c5 --beam 80 --estimator reference --no-cpu --steps 5 --warmup 3 --hash-slots $2 \
     --out gpurun_out/bi_c5_t$1_h$2.json > gpurun_out/bi_c5_t$1_h$2.log 2>&1
  grep -E "\] \[(reference|popcount)\] L=" gpurun_out/bi_c5_t$1_h$2.log | sed "s/^/c5 tag16=$1 hs=$2 /"
done
