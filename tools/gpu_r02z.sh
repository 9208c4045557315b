set -x
mkdir -p gpurun_out
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:beam_search -c 1 -o gpurun_out/prof_p1search_9M -f python tools/prof_donor.py 9000000 > gpurun_out/ncu_p1search.log 2>&1
tail -2 gpurun_out/ncu_p1search.log
