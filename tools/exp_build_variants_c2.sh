# A/B of construction knobs on the C2 bulk build (1M x 128): build.inserts_per_s of bench.py
set -x
for V in "" "$@"; do
  touch paper_2601_07048_b200/csrc/build.cu
  JB_NVCC_EXTRA="$V" python -m paper_2601_07048_b200._build > /dev/null
  for rep in 1 2; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --stream-rows 0 --beam 128 --estimator popcount --out gpurun_out/bv.json > /dev/null 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/bv.json')); print('VARIANT', repr(sys.argv[1]), 'build', d['build']['inserts_per_s'], d['build']['graph_sha'])" "$V"
  done
done
touch paper_2601_07048_b200/csrc/build.cu
