set -x
ncu --set full --import-source on --clock-control none -k regex:owner_merge_kernel --launch-skip 55 -c 1 -o gpurun_out/prof_owner_c4 python bench_configs.py c4 --total 5000000 --out gpurun_out/c4_ncu1.json > gpurun_out/ncu_owner_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:donor_scan_kernel --launch-skip 40 -c 1 -o gpurun_out/prof_donor_c4 python bench_configs.py c4 --total 5000000 --out gpurun_out/c4_ncu2.json > gpurun_out/ncu_donor_c4.log 2>&1
tail -3 gpurun_out/ncu_owner_c4.log gpurun_out/ncu_donor_c4.log
