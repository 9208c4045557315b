set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_build_gpu.py::test_config1_100k_build_identical_to_reference > gpurun_out/pytest_gpu_r02c.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu_r02c.log
bash profiles/profile_round.sh r02c --steps 10 --warmup 3
