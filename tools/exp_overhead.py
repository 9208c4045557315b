"""Per-call host overhead of search_knn_batch (tiny batches) on the bench index (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_07048_b200 as jb

x = jb.gen_lowrank(200_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
q = jb.gen_lowrank(10_000, 128, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
idx = jb.rabitq_fit(ds, bits=1, seed=1)
sp = jb.SearchParams(beam_width=128, k=10, rerank=True, estimator="popcount")
for nq in (1, 10, 100):
    qq = np.ascontiguousarray(q[:nq])
    for _ in range(20):
        jb.search_knn_batch(g, idx, qq, sp, exact_data=ds)
    ts = []
    for _ in range(200):
        t = time.perf_counter()
        jb.search_knn_batch(g, idx, qq, sp, exact_data=ds)
        ts.append(time.perf_counter() - t)
    print(f"nq={nq}: median {1e6 * np.median(ts):.1f} us per call", flush=True)
import cProfile, pstats
qq = np.ascontiguousarray(q[:10])
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    jb.search_knn_batch(g, idx, qq, sp, exact_data=ds)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
