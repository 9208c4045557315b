#!/bin/bash
# Run on the GPU box via gpurun: bench line + ncu launch list + one ncu --set full of the search kernel.
# Usage: bash profiles/profile_round.sh <tag> [extra bench args]
set -x
TAG=${1:-r01}; shift
mkdir -p gpurun_out
timeout 900 python bench.py "$@" --out gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.log
tail -5 gpurun_out/bench_${TAG}.log
L=$(python -c "import json;print(json.load(open('gpurun_out/bench_${TAG}.json'))['config']['beam_width'])")
EST=$(python -c "import json;print(json.load(open('gpurun_out/bench_${TAG}.json'))['config']['estimator'])")
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py "$@" --beam $L --estimator $EST --no-cpu --steps 3 --warmup 1 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
    -k regex:beam_search_kernel -c 1 -o gpurun_out/prof_search_${TAG} -f python bench.py "$@" --beam $L --estimator $EST --no-cpu \
    --steps 1 --warmup 1 > gpurun_out/ncu_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_${TAG}.log
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
    -k regex:rerank_kernel -c 1 -o gpurun_out/prof_rerank_${TAG} -f python bench.py "$@" --beam $L --estimator $EST --no-cpu \
    --steps 1 --warmup 1 > gpurun_out/ncu_rerank_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_rerank_${TAG}.log
ls -la gpurun_out
# per-launch DRAM traffic of the profiled search kernel -> bench.py's roofline.traffic
python - <<PY
import csv, io, json, subprocess
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", "gpurun_out/prof_search_${TAG}.ncu-rep", "--page", "raw",
      "--csv"], capture_output=True, text=True).stdout)))
h, u, r = raw[0], raw[1], raw[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
b = sum(float(r[h.index(m)].replace(",", "")) * scale[u[h.index(m)]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
bj = json.load(open("gpurun_out/bench_${TAG}.json"))
wl = bj["config"]["workload"] + f" L={bj['config']['beam_width']} {bj['config']['estimator']}"
json.dump({"workload": wl, "dram_bytes_per_launch": int(b), "source": "prof_search_${TAG}.ncu-rep (ncu --set full)"},
          open("gpurun_out/search_kernel_traffic.json", "w"), indent=1)
print("traffic", int(b))
PY
