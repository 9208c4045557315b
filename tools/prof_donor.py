"""Profile target for the connectivity repair's donor kernels (dev tool): bulk-build
N rows of DEEP-shaped 96-d data, then stream one 100K batch (whose repair runs the
donor seed / tensor-core screen / exact kernels).   python tools/prof_donor.py [N]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_07048_b200 as jb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_000
x = jb.gen_lowrank(n + 100_000, 96, seed=1, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
p = jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2, max_batch=100_000)
g = jb.GraphIndex(capacity=n + 100_000, degree_cap=32)
jb.insert_stream(g, ds, range(0, n), p)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
t0 = time.perf_counter()
jb.insert_stream(g, ds, range(n, n + 100_000), p)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(f"batch of 100K into {n}: {time.perf_counter() - t0:.3f} s", flush=True)
