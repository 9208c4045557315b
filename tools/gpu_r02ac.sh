set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_search_gpu.py tests/test_boundary_gpu.py -q -x > gpurun_out/pytest_r02ac.log 2>&1; echo rc=$?
tail -2 gpurun_out/pytest_r02ac.log
for S in 1 0; do for E in reference popcount; do
JB_SREC=$S timeout 600 python tools/prof_c3_search.py 64 $E 2>&1 | tail -1 | sed "s/^/SREC=$S /"
done; done
