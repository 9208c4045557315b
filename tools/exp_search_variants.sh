# A/B of search-kernel compile-time knobs on the GPU box (dev tool): for each
# JB_NVCC_EXTRA variant, rebuild search.cu and time the bench's search kernel.
#   bash tools/exp_search_variants.sh "-DJB_COOP_MAX=3" "-DJB_FAST_MINB=12" ...
set -x
mkdir -p gpurun_out
for V in "" "$@"; do
  touch paper_2601_07048_b200/csrc/search.cu
  JB_NVCC_EXTRA="$V" python -m paper_2601_07048_b200._build > /dev/null
  for EST in popcount reference; do
    timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --stream-rows 0 --beam 128 --estimator $EST \
      --out gpurun_out/var.json 2> /dev/null > /dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/var.json')); print('VARIANT', repr(sys.argv[1]), sys.argv[2], 'search_ms', d['kernel_ms']['search'], 'value', d['value'])" "$V" $EST
  done
done
touch paper_2601_07048_b200/csrc/search.cu
