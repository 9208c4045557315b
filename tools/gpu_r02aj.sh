set -x
mkdir -p gpurun_out
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:owner_merge_kernel" -c 2 -o gpurun_out/prof_owner_r02aj -f python tools/prof_donor.py 3000000 > /dev/null 2>&1
echo done
