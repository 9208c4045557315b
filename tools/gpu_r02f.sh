# Round 2 re-entry: GPU tests, bench (both estimators), full ncu with source of both search kernels.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_build_gpu.py::test_config1_100k_build_identical_to_reference > gpurun_out/pytest_gpu_r02f.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu_r02f.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --stream-rows 0 --out gpurun_out/bench_r02f.json 2> gpurun_out/bench_r02f.log; tail -3 gpurun_out/bench_r02f.log
for EST in popcount reference; do
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "kernel_alone/" \
    -k regex:beam_search_kernel -c 1 -o gpurun_out/prof_search_r02f_$EST -f python bench.py --beam 128 --estimator $EST --no-cpu \
    --stream-rows 0 --steps 1 --warmup 1 > gpurun_out/ncu_r02f_$EST.log 2>&1
tail -2 gpurun_out/ncu_r02f_$EST.log
done
