set -x
mkdir -p gpurun_out
timeout 1500 python bench_configs.py c3 --out gpurun_out/c3_r02bb.json > gpurun_out/c3_r02bb.log 2>&1; tail -1 gpurun_out/c3_r02bb.log | cut -c1-300
timeout 1500 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu --out gpurun_out/bench_c5_r02bb.json 2> gpurun_out/bench_c5_r02bb.log; tail -2 gpurun_out/bench_c5_r02bb.log
python -c "import json; d=json.load(open('gpurun_out/bench_c5_r02bb.json')); print('C5', d['value'], d['build']['inserts_per_s'], d['build']['search_kernel_roofline']['frac'])"
timeout 900 python bench_configs.py c1 --out gpurun_out/c1_r02bb.json > gpurun_out/c1_r02bb.log 2>&1; tail -1 gpurun_out/c1_r02bb.log | cut -c1-300
