set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | head -20 > gpurun_out/lscpu.txt; nproc >> gpurun_out/lscpu.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02a.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu_r02a.log
timeout 600 python bench.py --steps 10 --warmup 3 --out gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.log
tail -3 gpurun_out/bench_r02a.log
