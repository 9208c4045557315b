"""Streaming-insert phase profile at scale (dev tool): bulk-build N0 rows of a 96-d
low-rank set, then insert a few 100K batches with JB_PROFILE=1 phase timings."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_07048_b200 as jb

n0 = int(sys.argv[1]) if len(sys.argv) > 1 else 9_500_000
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 3
x = jb.gen_lowrank(n0 + nb * 100_000, 96, seed=1, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
ds.device()
p = jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2, max_batch=100_000)
g = jb.GraphIndex(ds.count, 32)
t = time.perf_counter()
jb.insert_stream(g, ds, range(0, n0), p)
torch.cuda.synchronize()
print(f"bulk {n0}: {time.perf_counter() - t:.2f} s", file=sys.stderr)
os.environ["JB_PROFILE"] = "1"
for i in range(nb):
    t = time.perf_counter()
    torch.cuda.nvtx.range_push("batch")
    jb.insert_stream(g, ds, range(n0 + i * 100_000, n0 + (i + 1) * 100_000), p)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print(f"batch {i}: {1e3 * (time.perf_counter() - t):.1f} ms", file=sys.stderr)
