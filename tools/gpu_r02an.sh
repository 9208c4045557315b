set -x
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
echo "== racecheck staged" > gpurun_out/sanitizer_racecheck_staged.log
timeout 1500 $CS --tool racecheck --racecheck-report analysis --print-limit 1000 python tools/sanitize_cases.py staged >> gpurun_out/sanitizer_racecheck_staged.log 2>&1
echo "rc=$?" >> gpurun_out/sanitizer_racecheck_staged.log
grep -E "RACECHECK SUMMARY" gpurun_out/sanitizer_racecheck_staged.log
grep -E "^========= (Error|Warning): Race" gpurun_out/sanitizer_racecheck_staged.log | sed 's/+0x[0-9a-f]*//g' | sort | uniq -c
timeout 900 python -m pytest tests/test_build_gpu.py -q -x --deselect tests/test_build_gpu.py::test_config1_100k_build_identical_to_reference 2>&1 | tail -1
timeout 600 python tools/insert_search_roofline.py 3000000 2>&1 | tail -1
timeout 900 python tools/insert_search_roofline.py 9000000 2>&1 | tail -1
