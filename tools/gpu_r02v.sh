set -x
mkdir -p gpurun_out
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:beam_search -c 1 -o gpurun_out/prof_c3_search_r02v -f python tools/prof_c3_search.py 64 reference > gpurun_out/ncu_c3_r02v.log 2>&1
tail -2 gpurun_out/ncu_c3_r02v.log
bash profiles/profile_round.sh r02v_c5 --config c5 --steps 10 --warmup 3
