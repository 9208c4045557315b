set -x
mkdir -p gpurun_out
bash tools/sanitize.sh
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --stream-rows 0 --out gpurun_out/bench_r02e.json 2> gpurun_out/bench_r02e.log; tail -3 gpurun_out/bench_r02e.log
timeout 1500 python bench.py --config c5 --steps 10 --warmup 3 --out gpurun_out/bench_c5_r02e.json 2> gpurun_out/bench_c5_r02e.log; tail -5 gpurun_out/bench_c5_r02e.log
