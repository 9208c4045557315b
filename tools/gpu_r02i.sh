# tensor-core donor screen: parity + repair-heavy build tests
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_donor_tc_gpu.py -q -x > gpurun_out/pytest_r02i.log 2>&1; echo rc=$?
tail -30 gpurun_out/pytest_r02i.log
timeout 900 python -m pytest tests/test_build_gpu.py -q -x --deselect tests/test_build_gpu.py::test_config1_100k_build_identical_to_reference > gpurun_out/pytest_r02i_build.log 2>&1; echo rc=$?
tail -5 gpurun_out/pytest_r02i_build.log
