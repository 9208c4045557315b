#!/bin/bash
# compute-sanitizer over the round-2 re-entry paths (screen case)
mkdir -p gpurun_out
python -m paper_2601_07048_b200._build > /dev/null 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python tools/sanitize_cases.py screen 2>&1 | tail -1
for tool in memcheck synccheck initcheck; do
  echo "== $tool (screen case)" > gpurun_out/sanitizer_${tool}_screen.log
  timeout 900 $CS --tool $tool --print-limit 200 --error-exitcode 9 python tools/sanitize_cases.py screen >> gpurun_out/sanitizer_${tool}_screen.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_${tool}_screen.log
  tail -3 gpurun_out/sanitizer_${tool}_screen.log
done
echo "== racecheck screen" > gpurun_out/sanitizer_racecheck_screen.log
timeout 1200 $CS --tool racecheck --racecheck-report analysis --print-limit 1000 python tools/sanitize_cases.py screen >> gpurun_out/sanitizer_racecheck_screen.log 2>&1
echo "rc=$?" >> gpurun_out/sanitizer_racecheck_screen.log
tail -3 gpurun_out/sanitizer_racecheck_screen.log
grep -c "Race reported" gpurun_out/sanitizer_racecheck_screen.log
grep -E "at .*search.cu:[0-9]+|at .*build.cu:[0-9]+|at .*screen.cu:[0-9]+" gpurun_out/sanitizer_racecheck_screen.log | sed -E 's/.*(search|build|screen)\.cu:([0-9]+).*/\1.cu:\2/' | sort | uniq -c | head -20
