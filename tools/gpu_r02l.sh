set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_donor_tc_gpu.py -q -x 2>&1 | tail -3
JB_PROFILE=1 timeout 600 python tools/prof_donor.py 3000000 > gpurun_out/prof_donor_plain_m.log 2>&1; grep "scan\|batch of" gpurun_out/prof_donor_plain_l.log | tail -4
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:donor_screen -c 1 -o gpurun_out/prof_donor_r02m -f python tools/prof_donor.py 3000000 > gpurun_out/ncu_donor_r02m.log 2>&1
tail -2 gpurun_out/ncu_donor_r02m.log
