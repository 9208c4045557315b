set -x
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/launches_batch3M.csv python tools/prof_donor.py 3000000 > /dev/null 2>&1
echo done
