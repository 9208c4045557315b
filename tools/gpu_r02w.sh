set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_search_gpu.py tests/test_boundary_gpu.py tests/test_rabitq_props.py -q -x > gpurun_out/pytest_r02w.log 2>&1; echo rc=$?
tail -2 gpurun_out/pytest_r02w.log
timeout 600 python tools/prof_c3_search.py 64 reference 2>&1 | tail -1
for HS in 0 1024 2048; do
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu --stream-rows 0 --beam 80 --estimator reference --hash-slots $HS --out gpurun_out/c5_hs$HS.json 2> gpurun_out/c5_hs$HS.log
python -c "import json; d=json.load(open('gpurun_out/c5_hs$HS.json')); print('HS $HS', d['value'], d['kernel_ms']['search'], d['per_query'])"
done
