set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r02ba.log 2>&1; echo rc=$?
tail -1 gpurun_out/pytest_r02ba.log
bash tools/gpu_r02az.sh
