set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_build_gpu.py tests/test_donor_tc_gpu.py -q -x > gpurun_out/pytest_r02ar.log 2>&1; echo rc=$?
tail -1 gpurun_out/pytest_r02ar.log
JB_PROFILE=1 timeout 900 python bench_configs.py c4 --out gpurun_out/c4_r02ar.json > gpurun_out/c4_r02ar.log 2> gpurun_out/c4_r02ar.err; tail -1 gpurun_out/c4_r02ar.log
grep "batch \[9900000" gpurun_out/c4_r02ar.err
grep -c "no evictions" gpurun_out/c4_r02ar.err
grep -c "repair round 1:" gpurun_out/c4_r02ar.err
