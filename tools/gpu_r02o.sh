# config matrix: C2 on the reference's iid Gaussian rows, C3 d_int=32 at R=64, ncu of the C3 search kernel
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --data gaussian --steps 5 --warmup 3 --stream-rows 0 --out gpurun_out/bench_c2_gauss_r02o.json 2> gpurun_out/bench_c2_gauss_r02o.log; tail -3 gpurun_out/bench_c2_gauss_r02o.log
timeout 1500 python bench_configs.py c3 --dint 32 --R 64 --lbuild 128 --out gpurun_out/c3_dint32_R64_r02o.json > gpurun_out/c3_R64_r02o.log 2>&1; tail -2 gpurun_out/c3_R64_r02o.log
