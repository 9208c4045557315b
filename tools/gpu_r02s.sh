set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_build_gpu.py tests/test_donor_tc_gpu.py -q -x --deselect tests/test_build_gpu.py::test_config1_100k_build_identical_to_reference > gpurun_out/pytest_r02t.log 2>&1; echo rc=$?
tail -2 gpurun_out/pytest_r02t.log
JB_PROFILE=1 timeout 900 python bench_configs.py c4 --out gpurun_out/c4_r02t.json > gpurun_out/c4_r02t.log 2> gpurun_out/c4_r02t.err; echo rc=$?
tail -2 gpurun_out/c4_r02t.log
grep "batch \[9900000" gpurun_out/c4_r02t.err
grep "repair timings" gpurun_out/c4_r02t.err | tail -2
grep "tensor-core donor" gpurun_out/c4_r02t.err | awk "{s+=\$5} END {print \"redo rows total\", s}"
