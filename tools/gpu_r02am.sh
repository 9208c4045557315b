set -x
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for c in insert pipeline staged; do
  echo "== racecheck $c" > gpurun_out/sanitizer_racecheck_$c.log
  timeout 1500 $CS --tool racecheck --racecheck-report analysis --print-limit 1000 python tools/sanitize_cases.py $c >> gpurun_out/sanitizer_racecheck_$c.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_racecheck_$c.log
  grep -E "RACECHECK SUMMARY|in build.cu|in donor_tc|in search.cu|in common" gpurun_out/sanitizer_racecheck_$c.log | sort | uniq -c | head -12
done
