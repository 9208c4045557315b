set -x
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_full_r02aq.log 2>&1; echo rc=$?
tail -1 gpurun_out/pytest_full_r02aq.log
JB_PROFILE=1 timeout 900 python bench_configs.py c4 --out gpurun_out/c4_r02aq.json > gpurun_out/c4_r02aq.log 2> gpurun_out/c4_r02aq.err; tail -1 gpurun_out/c4_r02aq.log
grep "batch \[9900000" gpurun_out/c4_r02aq.err
