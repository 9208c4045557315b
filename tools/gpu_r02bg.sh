set -x
timeout 900 python -m pytest tests/test_search_gpu.py tests/test_boundary_gpu.py tests/test_rabitq_props.py -q -x 2>&1 | tail -1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_call2.csv python tools/prof_c3_search.py 64 reference > /dev/null 2>&1
grep rotate_gemm gpurun_out/launches_c3_call2.csv | head -2 | cut -c1-40,300-400
timeout 600 python tools/prof_c3_search.py 64 reference 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --stream-rows 0 --beam 128 --out gpurun_out/bv.json > /dev/null 2>&1
python -c "import json; d=json.load(open('gpurun_out/bv.json')); print('C2', d['value'], d['kernel_ms'])"
