#!/bin/bash
# compute-sanitizer pass over the product kernels (run on the GPU box via gpurun).
# memcheck / synccheck / initcheck over all cases; racecheck per case in analysis
# mode (one report per hazard site). Logs: gpurun_out/sanitizer_<tool>[_case].log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck; do
  echo "== $tool" > gpurun_out/sanitizer_$tool.log
  timeout 1500 $CS --tool $tool --print-limit 200 --error-exitcode 9 \
      python tools/sanitize_cases.py >> gpurun_out/sanitizer_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_$tool.log
  tail -3 gpurun_out/sanitizer_$tool.log
done
for c in search insert pipeline protocol; do
  echo "== racecheck $c" > gpurun_out/sanitizer_racecheck_$c.log
  timeout 1500 $CS --tool racecheck --racecheck-report analysis --print-limit 1000 \
      python tools/sanitize_cases.py $c >> gpurun_out/sanitizer_racecheck_$c.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_racecheck_$c.log
  tail -3 gpurun_out/sanitizer_racecheck_$c.log
done
