set -x
for C in 0 3334 2500 2000; do
JB_DEVICE_CHUNK=$C timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --stream-rows 0 --beam 128 --estimator popcount --out gpurun_out/chunk$C.json 2>/dev/null >/dev/null
python -c "import json; d=json.load(open('gpurun_out/chunk$C.json')); print('CHUNK $C', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
