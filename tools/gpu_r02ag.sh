set -x
touch paper_2601_07048_b200/csrc/build.cu
JB_NVCC_EXTRA="-DJB_OWNER_STATS" python -m paper_2601_07048_b200._build > /dev/null
timeout 600 python tools/exp_owner_stats.py 3000000 2>&1 | tail -4
touch paper_2601_07048_b200/csrc/build.cu
