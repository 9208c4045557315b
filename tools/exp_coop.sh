set -x
for c in 2 6 8; do
  touch paper_2601_07048_b200/csrc/search.cu && JB_NVCC_EXTRA=-DJB_COOP_MAX=$c python -m paper_2601_07048_b200._build > /dev/null
  echo "COOP_MAX=$c"; timeout 300 python tools/exp_search.py 128 2>&1 | grep "hash     0"
done
touch paper_2601_07048_b200/csrc/search.cu && python -m paper_2601_07048_b200._build > /dev/null
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 2> gpurun_out/ref_arm.log | tail -1
