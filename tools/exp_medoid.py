"""Medoid / column-mean kernel timing (dev tool): jb.medoid on n x d low-rank rows."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_07048_b200 as jb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
x = jb.gen_lowrank(n, d, seed=1, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
ds.device()
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    m = jb.medoid(ds)
    torch.cuda.synchronize()
    print(f"medoid {n}x{d}: {1e3 * (time.perf_counter() - t):.2f} ms -> {m}", file=sys.stderr)
