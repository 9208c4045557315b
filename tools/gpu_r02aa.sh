set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_search_gpu.py tests/test_build_gpu.py tests/test_knn_gpu.py -q -x --deselect tests/test_build_gpu.py::test_config1_100k_build_identical_to_reference > gpurun_out/pytest_r02ab.log 2>&1; echo rc=$?
tail -2 gpurun_out/pytest_r02ab.log
JB_PROFILE=1 timeout 900 python bench_configs.py c4 --out gpurun_out/c4_r02ab.json > gpurun_out/c4_r02ab.log 2> gpurun_out/c4_r02ab.err; echo rc=$?
tail -1 gpurun_out/c4_r02ab.log
grep "batch \[9900000" gpurun_out/c4_r02ab.err
timeout 900 python bench_configs.py c1 --out gpurun_out/c1_r02ab.json > gpurun_out/c1_r02ab.log 2>&1; tail -1 gpurun_out/c1_r02ab.log | cut -c1-600
