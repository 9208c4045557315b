"""Build the same data twice (and once more in streaming batches) and compare graphs (dev tool)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_07048_b200 as jb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 96
x = jb.gen_lowrank(n, d, seed=1, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
p = jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2, max_batch=100_000)
hs = []
for rep in range(3):
    g = jb.build(ds, p)
    torch.cuda.synchronize()
    adj = g.adjacency[:n]
    h = hashlib.sha1(adj.tobytes()).hexdigest()[:12]
    hs.append(adj.copy())
    print(f"rep {rep}: sha1 {h} entry {g.entry_point} bridges_last {g.last_bridges}", flush=True)
for r in (1, 2):
    diff = np.nonzero((hs[0] != hs[r]).any(axis=1))[0]
    print(f"rep 0 vs {r}: {diff.size} rows differ; first {diff[:10].tolist()}", flush=True)
