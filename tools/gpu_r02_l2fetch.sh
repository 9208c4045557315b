#!/bin/bash
# L2 fetch granularity (cudaLimitMaxL2FetchGranularity) vs search kernel time / DRAM bytes
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
for v in 0 32 64; do  # (JB_L2_FETCH hook removed after this experiment; see DESIGN 9b)
  JB_L2_FETCH=$v timeout 600 python bench.py --config c5 --beam 80 --estimator reference --no-cpu --steps 5 --warmup 3 \
     --out gpurun_out/l2f_c5_$v.json > gpurun_out/l2f_c5_$v.log 2>&1
  python -c "import json;b=json.load(open('gpurun_out/l2f_c5_$v.json'));print('c5 fetch $v', b['value'], b['kernel_ms'])"
done
for v in 0 64; do
  JB_L2_FETCH=$v timeout 600 python bench.py --beam 128 --no-cpu --steps 5 --warmup 3 \
     --out gpurun_out/l2f_c2_$v.json > gpurun_out/l2f_c2_$v.log 2>&1
  python -c "import json;b=json.load(open('gpurun_out/l2f_c2_$v.json'));print('c2 fetch $v', b['value'], b['kernel_ms'], b['estimators'])"
done
for v in 0 64; do
  JB_L2_FETCH=$v timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none \
     --nvtx --nvtx-include "kernel_alone/" -k regex:beam_search_kernel -c 1 --csv python bench.py --config c5 --beam 80 \
     --estimator reference --no-cpu --steps 1 --warmup 1 2>/dev/null | grep -E "dram__bytes|duration|hit_rate" | cut -c1-400
done
