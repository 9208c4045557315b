# C4 streaming with the tensor-core donor screen (JB_PROFILE phase timings), C3 at d_int=32
set -x
mkdir -p gpurun_out
JB_PROFILE=1 timeout 900 python bench_configs.py c4 --out gpurun_out/c4_r02j.json > gpurun_out/c4_r02j.log 2> gpurun_out/c4_r02j.err; echo rc=$?
tail -3 gpurun_out/c4_r02j.log
grep -c "tensor-core donor" gpurun_out/c4_r02j.err
timeout 1200 python bench_configs.py c3 --dint 32 --out gpurun_out/c3_dint32_r02j.json > gpurun_out/c3_r02j.log 2>&1; echo rc=$?
tail -3 gpurun_out/c3_r02j.log
