set -x
mkdir -p gpurun_out
JB_PROFILE=1 timeout 600 python tools/prof_donor.py 3000000 > gpurun_out/prof_donor_plain.log 2>&1; tail -12 gpurun_out/prof_donor_plain.log
timeout 1200 ncu --profile-from-start off --set full --import-source on -k regex:donor -c 6 -o gpurun_out/prof_donor_r02k -f python tools/prof_donor.py 3000000 > gpurun_out/ncu_donor_r02k.log 2>&1
tail -3 gpurun_out/ncu_donor_r02k.log
