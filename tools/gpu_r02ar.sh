set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_build_gpu.py tests/test_donor_tc_gpu.py -q -x > gpurun_out/pytest_r02ax.log 2>&1; echo rc=$?
tail -1 gpurun_out/pytest_r02ax.log
JB_PROFILE=1 timeout 900 python bench_configs.py c4 --out gpurun_out/c4_r02ax.json > gpurun_out/c4_r02ax.log 2> gpurun_out/c4_r02ax.err; tail -1 gpurun_out/c4_r02ax.log
grep "batch \[9900000" gpurun_out/c4_r02ax.err
grep -c "no evictions" gpurun_out/c4_r02ax.err
grep -c "repair round 1:" gpurun_out/c4_r02ax.err
