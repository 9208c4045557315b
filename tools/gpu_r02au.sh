set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_build_gpu.py -q -x --deselect tests/test_build_gpu.py::test_config1_100k_build_identical_to_reference > gpurun_out/pytest_r02au.log 2>&1; echo rc=$?
tail -1 gpurun_out/pytest_r02au.log
for i in 1 2; do JB_PROFILE=1 timeout 600 python tools/prof_donor.py 3000000 2>&1 | grep "batch \[3000000"; done
