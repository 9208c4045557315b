timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_call.csv python tools/prof_c3_search.py 64 reference > /dev/null 2>&1
echo done
