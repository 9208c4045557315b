set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r02aw.log 2>&1; echo rc=$?
tail -3 gpurun_out/pytest_r02aw.log
for C in 1 0; do JB_CLOSURE=$C JB_PROFILE=1 timeout 600 python tools/prof_donor.py 3000000 2>&1 | grep "batch \[3000000" | sed "s/^/CLOSURE=$C /"; done
