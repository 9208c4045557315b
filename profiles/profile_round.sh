#!/bin/bash
# Run on the GPU box via gpurun: bench line + ncu launch list + one ncu --set full of the search kernel.
# Usage: bash profiles/profile_round.sh <tag> [extra bench args]
# The --set full capture is of the 10K-query search launch that bench.py's kernel_ms times
# (NVTX range "kernel_alone"), so `traffic` and the instruction count are per that launch.
set -x
TAG=${1:-r02}; shift
mkdir -p gpurun_out
timeout 900 python bench.py "$@" --out gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.log
tail -5 gpurun_out/bench_${TAG}.log
L=$(python -c "import json;print(json.load(open('gpurun_out/bench_${TAG}.json'))['config']['beam_width'])")
EST=$(python -c "import json;print(json.load(open('gpurun_out/bench_${TAG}.json'))['estimator'])")
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py "$@" --beam $L --estimator $EST --no-cpu --steps 3 --warmup 1 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "kernel_alone/" \
    -k regex:beam_search_kernel -c 1 -o gpurun_out/prof_search_${TAG} -f python bench.py "$@" --beam $L --estimator $EST --no-cpu \
    --steps 1 --warmup 1 > gpurun_out/ncu_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_${TAG}.log
ls -la gpurun_out
# per-launch DRAM traffic + warp instructions of the profiled search launch -> bench.py's roofline
python - <<PY
import csv, io, json, subprocess
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", "gpurun_out/prof_search_${TAG}.ncu-rep", "--page", "raw",
      "--csv"], capture_output=True, text=True).stdout)))
h, u, r = raw[0], raw[1], raw[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9,
         "": 1}
val = lambda m: float(r[h.index(m)].replace(",", "")) * scale.get(u[h.index(m)], 1)
b = sum(val(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
inst = val("smsp__inst_executed.sum")
grid = r[h.index("launch__grid_size")] if "launch__grid_size" in h else None
bj = json.load(open("gpurun_out/bench_${TAG}.json"))
wl = bj["config"]["workload"] + f" L={bj['config']['beam_width']} {bj['estimator']}"
json.dump({"workload": wl, "dram_bytes_per_launch": int(b), "warp_inst_per_launch": int(inst), "grid": grid,
           "queries_per_launch": 10000, "source": "prof_search_${TAG}.ncu-rep (ncu --set full, NVTX kernel_alone)"},
          open("gpurun_out/search_kernel_traffic.json", "w"), indent=1)
print("traffic", int(b), "inst", int(inst))
PY
