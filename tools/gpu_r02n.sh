set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_donor_tc_gpu.py -q -x 2>&1 | tail -2
JB_PROFILE=1 timeout 600 python tools/prof_donor.py 3000000 > gpurun_out/prof_donor_plain_n.log 2>&1; grep "scan\|batch of" gpurun_out/prof_donor_plain_n.log | tail -3
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/launches_c4batch_9M.csv python tools/prof_donor.py 9000000 > gpurun_out/ncu_c4batch.log 2>&1
tail -2 gpurun_out/ncu_c4batch.log
