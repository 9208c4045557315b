set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 --out gpurun_out/bench_r02ao.json 2> gpurun_out/bench_r02ao.log; tail -2 gpurun_out/bench_r02ao.log
python -c "import json; d=json.load(open('gpurun_out/bench_r02ao.json')); print(d['value'], d['e2e']['value'], d['build']['inserts_per_s'], d['build']['search_kernel_roofline'], d['cpu_baseline'])"
timeout 1500 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu --out gpurun_out/bench_c5_r02ao.json 2> gpurun_out/bench_c5_r02ao.log; tail -2 gpurun_out/bench_c5_r02ao.log
python -c "import json; d=json.load(open('gpurun_out/bench_c5_r02ao.json')); print(d['value'], d['build']['inserts_per_s'], d['build']['search_kernel_roofline'])"
