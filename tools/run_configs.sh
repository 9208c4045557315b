#!/bin/bash
# Secondary BASELINE.json configs on one B200 (bench_configs.py); JSON lines -> gpurun_out/
mkdir -p gpurun_out
for c in "$@"; do
  timeout 1500 python bench_configs.py $c --out gpurun_out/config_$c.json > gpurun_out/config_$c.log 2>&1
  echo "$c rc=$?"; tail -2 gpurun_out/config_$c.log
done
