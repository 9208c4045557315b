set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_search_gpu.py tests/test_build_gpu.py tests/test_knn_gpu.py tests/test_boundary_gpu.py -q -x --deselect tests/test_build_gpu.py::test_config1_100k_build_identical_to_reference > gpurun_out/pytest_r02ap.log 2>&1; echo rc=$?
tail -1 gpurun_out/pytest_r02ap.log
timeout 600 python tools/insert_search_roofline.py 9000000 2>&1 | tail -1
timeout 900 python bench_configs.py c1 --out gpurun_out/c1_r02ap.json 2>&1 | tail -1 | cut -c1-400
JB_PROFILE=1 timeout 900 python bench_configs.py c4 --out gpurun_out/c4_r02ap.json > gpurun_out/c4_r02ap.log 2> gpurun_out/c4_r02ap.err; tail -1 gpurun_out/c4_r02ap.log
grep "batch \[9900000" gpurun_out/c4_r02ap.err
