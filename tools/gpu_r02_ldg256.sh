#!/bin/bash
# 256-bit record loads: parity + C5 / C2 search kernel time + C5 DRAM bytes
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_search_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py --config c5 --beam 80 --estimator reference --no-cpu --steps 5 --warmup 3 \
     --out gpurun_out/ldg_c5.json > gpurun_out/ldg_c5.log 2>&1
python -c "import json;b=json.load(open('gpurun_out/ldg_c5.json'));print('c5', b['value'], b['kernel_ms'], b['recall_at_10'])"
timeout 600 python bench.py --beam 128 --no-cpu --steps 5 --warmup 3 --out gpurun_out/ldg_c2.json > gpurun_out/ldg_c2.log 2>&1
python -c "import json;b=json.load(open('gpurun_out/ldg_c2.json'));print('c2', b['value'], b['kernel_ms'], b['estimators'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__m_xbar2l1tex_read_sectors_mem_lg_op_ld.sum --clock-control none \
     --nvtx --nvtx-include "kernel_alone/" -k regex:beam_search_kernel -c 1 --csv python bench.py --config c5 --beam 80 \
     --estimator reference --no-cpu --steps 1 --warmup 1 2>/dev/null | grep -E "beam_search" | awk -F'","' '{print $(NF-2), $NF}'
