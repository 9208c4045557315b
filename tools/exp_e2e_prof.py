import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2601_07048_b200 as jb
from paper_2601_07048_b200 import search as js
x = jb.gen_lowrank(1_000_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
q = jb.gen_lowrank(10_000, 128, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
idx = jb.rabitq_fit(ds, bits=1, seed=1)
sp = jb.SearchParams(beam_width=128, k=10, rerank=True, estimator="popcount")
for chunk in (10000, 5000, 2500):
    js.PIPELINE["chunk"] = chunk
    for _ in range(3): jb.search_knn_batch(g, idx, q, sp, exact_data=ds)
    os.environ["JB_PIPE_PROFILE"] = "1"
    for _ in range(4):
        t = time.perf_counter(); jb.search_knn_batch(g, idx, q, sp, exact_data=ds); print(f"chunk {chunk} call {1e3*(time.perf_counter()-t):.3f} ms", file=sys.stderr, flush=True)
    del os.environ["JB_PIPE_PROFILE"]
