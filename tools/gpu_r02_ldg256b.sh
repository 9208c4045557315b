#!/bin/bash
# A/B: 256-bit load of the m=1 float-estimator records (JB_LDG256_R1), C2 both estimators
mkdir -p gpurun_out
for v in 1 0 1 0; do
  touch paper_2601_07048_b200/csrc/search.cu
  JB_NVCC_EXTRA="-DJB_LDG256_R1=$v" python -m paper_2601_07048_b200._build > /dev/null 2>&1
  timeout 600 python bench.py --beam 128 --no-cpu --steps 5 --warmup 3 --out gpurun_out/ldgb_$v.json > /dev/null 2>&1
  python -c "import json;b=json.load(open('gpurun_out/ldgb_$v.json'));e=b['estimators'];print('R1=$v ref', e['reference']['search_kernel_ms'], 'pop', e['popcount']['search_kernel_ms'])"
done
touch paper_2601_07048_b200/csrc/search.cu
