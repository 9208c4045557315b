set -x
mkdir -p gpurun_out
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:owner_merge|phase2_kernel" -c 2 -o gpurun_out/prof_merge_r02q -f python tools/prof_donor.py 3000000 > gpurun_out/ncu_merge_r02q.log 2>&1
tail -2 gpurun_out/ncu_merge_r02q.log
