set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_build_gpu.py tests/test_donor_tc_gpu.py -q -x --deselect tests/test_build_gpu.py::test_config1_100k_build_identical_to_reference > gpurun_out/pytest_r02ah.log 2>&1; echo rc=$?
tail -2 gpurun_out/pytest_r02ah.log
JB_PROFILE=1 timeout 600 python tools/prof_donor.py 3000000 2>&1 | grep "batch \[3000000\|batch of"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --stream-rows 0 --beam 128 --estimator popcount --out gpurun_out/bv.json > /dev/null 2>&1
python -c "import json; d=json.load(open('gpurun_out/bv.json')); print('C2 build', d['build']['inserts_per_s'], d['build']['graph_sha'])"
