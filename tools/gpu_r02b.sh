set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02b.log 2>&1; echo build rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02b.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu_r02b.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 --out gpurun_out/ref_r02b.json 2> gpurun_out/ref_r02b.log; echo ref rc=$?
tail -4 gpurun_out/ref_r02b.log
bash profiles/profile_round.sh r02b --steps 10 --warmup 3
