set -x
mkdir -p gpurun_out
JB_PROFILE=1 timeout 900 python bench_configs.py c4 --out gpurun_out/c4_r02r.json > gpurun_out/c4_r02r.log 2> gpurun_out/c4_r02r.err; echo rc=$?
tail -2 gpurun_out/c4_r02r.log
grep "batch \[9900000" gpurun_out/c4_r02r.err
