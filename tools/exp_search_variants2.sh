# A/B of search compile knobs on the insert-path (exact, HBM) search kernel and the C2 headline
set -x
for V in "" "$@"; do
  touch paper_2601_07048_b200/csrc/search.cu
  JB_NVCC_EXTRA="$V" python -m paper_2601_07048_b200._build > /dev/null
  timeout 600 python tools/insert_search_roofline.py 3000000 2>&1 | tail -1 | sed "s/^/VARIANT '$V' /"
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --stream-rows 0 --beam 128 --estimator popcount --out gpurun_out/var.json > /dev/null 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/var.json')); print('VARIANT', repr(sys.argv[1]), 'c2 search_ms', d['kernel_ms']['search'], 'value', d['value'], 'build', d['build']['inserts_per_s'])" "$V"
done
touch paper_2601_07048_b200/csrc/search.cu
