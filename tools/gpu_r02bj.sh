#!/bin/bash
# 1M x 128 bulk build: per-batch phase profile and per-kernel launch durations
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
JB_EXP_PROFILE=1 JB_EXP_REPS=2 timeout 600 python tools/exp_build_prof.py > gpurun_out/bj_prof.log 2>&1
tail -60 gpurun_out/bj_prof.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bj_launches.csv \
   python tools/exp_build_prof.py > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/bj_launches.csv")))
h = None; agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if h is None:
        if "Kernel Name" in r: h = r
        continue
    if len(r) != len(h) or r[h.index("Metric Name")] != "gpu__time_duration.sum": continue
    name = r[h.index("Kernel Name")].split("(")[0][:90]
    v = float(r[h.index("Metric Value")].replace(",", ""))
    unit = r[h.index("Metric Unit")]
    v = v / 1000.0 if unit == "nsecond" else (v if unit == "usecond" else v * 1000.0)
    agg[name][0] += 1; agg[name][1] += v
tot = sum(a[1] for a in agg.values())
print("total kernel us (both builds: warm-up 250K + 1M)", round(tot))
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{t:10.0f} us {n:5d}  {k}")
PY
