set -x
mkdir -p gpurun_out
BENCH_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --stream-rows 0 --beam 128 --out gpurun_out/bench_n2_r02at.json > gpurun_out/bench_n2_r02at.log 2>&1; echo rc=$?
tail -3 gpurun_out/bench_n2_r02at.log | cut -c1-600
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/ref_n2_r02at.log 2>&1; echo rc=$?
tail -2 gpurun_out/ref_n2_r02at.log | cut -c1-300
