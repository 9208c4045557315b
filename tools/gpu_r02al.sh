set -x
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python tools/sanitize_cases.py staged 2>&1 | tail -2
for tool in memcheck synccheck initcheck; do
  echo "== $tool staged" > gpurun_out/sanitizer_${tool}_staged.log
  timeout 1500 $CS --tool $tool --print-limit 200 --error-exitcode 9 python tools/sanitize_cases.py staged >> gpurun_out/sanitizer_${tool}_staged.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_${tool}_staged.log
  tail -4 gpurun_out/sanitizer_${tool}_staged.log
done
