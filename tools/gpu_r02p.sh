# Gram-screened owner-merge prune: parity + A/B timing
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_build_gpu.py tests/test_donor_tc_gpu.py -q -x --deselect tests/test_build_gpu.py::test_config1_100k_build_identical_to_reference > gpurun_out/pytest_r02p.log 2>&1; echo rc=$?
tail -3 gpurun_out/pytest_r02p.log
for G in 1; do
JB_PROFILE=1 timeout 600 python tools/prof_donor.py 3000000 > gpurun_out/prof_gram$G.log 2>&1; grep "batch \[3000000\|batch of" gpurun_out/prof_gram$G.log | tail -2
done
JB_OWNER_DEFER=0 JB_PROFILE=1 timeout 600 python tools/prof_donor.py 3000000 > gpurun_out/prof_nodefer.log 2>&1; grep "batch \[3000000\|batch of" gpurun_out/prof_nodefer.log | tail -2
