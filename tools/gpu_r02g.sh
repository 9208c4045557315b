# screened bit-exact estimator: parity tests + A/B kernel time
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_search_gpu.py tests/test_boundary_gpu.py tests/test_knn_gpu.py -q -x > gpurun_out/pytest_r02g.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_r02g.log
for S in 1 0; do
JB_SCREEN=$S timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --stream-rows 0 --estimator reference --beam 128 --out gpurun_out/bench_r02g_s$S.json 2> gpurun_out/bench_r02g_s$S.log; tail -2 gpurun_out/bench_r02g_s$S.log
done
