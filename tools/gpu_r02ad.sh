set -x
mkdir -p gpurun_out
timeout 1500 python bench_configs.py c3 --out gpurun_out/c3_r02ad.json > gpurun_out/c3_r02ad.log 2>&1; tail -1 gpurun_out/c3_r02ad.log | cut -c1-1500
timeout 1500 python bench_configs.py c3 --dint 32 --R 64 --lbuild 128 --out gpurun_out/c3_dint32_R64_r02ad.json > gpurun_out/c3b_r02ad.log 2>&1; tail -1 gpurun_out/c3b_r02ad.log | cut -c1-300
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:beam_search -c 1 -o gpurun_out/prof_c3_search_r02ad -f python tools/prof_c3_search.py 64 reference > gpurun_out/ncu_c3_r02ad.log 2>&1
tail -1 gpurun_out/ncu_c3_r02ad.log
