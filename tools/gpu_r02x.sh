set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_search_gpu.py tests/test_boundary_gpu.py tests/test_rabitq_props.py -q -x > gpurun_out/pytest_r02x.log 2>&1; echo rc=$?
tail -2 gpurun_out/pytest_r02x.log
timeout 600 python tools/prof_c3_search.py 64 reference 2>&1 | tail -1
timeout 600 python tools/prof_c3_search.py 64 popcount 2>&1 | tail -1
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu --stream-rows 0 --beam 80 --out gpurun_out/c5_r02x.json 2> gpurun_out/c5_r02x.log
tail -3 gpurun_out/c5_r02x.log
