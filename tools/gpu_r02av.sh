set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_search_gpu.py tests/test_boundary_gpu.py -q -x > gpurun_out/pytest_r02av.log 2>&1; echo rc=$?
tail -1 gpurun_out/pytest_r02av.log
for i in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --stream-rows 0 --beam 128 --out gpurun_out/bv.json > /dev/null 2>&1
python -c "import json; d=json.load(open('gpurun_out/bv.json')); print('C2', d['value'], d['kernel_ms']['search'], d['estimators'])"
done
