set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02d.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu_r02d.log
