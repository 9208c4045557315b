"""Streaming-path determinism across processes: insert_stream from an empty graph (seed batch of
max_batch rows) then 100K batches; prints the adjacency hash (dev tool)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_07048_b200 as jb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 500_000
mb = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000
x = jb.gen_lowrank(n, 96, seed=1, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
p = jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2, max_batch=mb)
g = jb.GraphIndex(n, 32)
jb.insert_stream(g, ds, range(0, n), p)
torch.cuda.synchronize()
print(f"stream n={n} mb={mb}: sha1 {hashlib.sha1(g.adjacency[:n].tobytes()).hexdigest()[:12]} entry {g.entry_point}")
g2 = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2, max_batch=100_000))
print(f"build n={n}: sha1 {hashlib.sha1(g2.adjacency[:n].tobytes()).hexdigest()[:12]} entry {g2.entry_point}")
