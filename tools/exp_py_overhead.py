"""Python-side cost of one search_knn_batch call, piece by piece (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2601_07048_b200 as jb
from paper_2601_07048_b200 import search as js

x = jb.gen_lowrank(200_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
idx = jb.rabitq_fit(ds, bits=1, seed=1)
sp = jb.SearchParams(beam_width=128, k=10, rerank=True, estimator="popcount")
q = np.zeros((10_000, 128), np.float32)


def t(fn, n=200):
    fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return 1e6 * (time.perf_counter() - t0) / n


print(f"_host_results {t(lambda: js._host_results(10_000, 10)):.1f} us")
print(f"_knn_plan     {t(lambda: js._knn_plan(g, idx, 128, sp, ds)):.1f} us")
print(f"as_graph+validate {t(lambda: js._validate(js.as_graph(g), 128)):.1f} us")
print(f"asarray       {t(lambda: np.ascontiguousarray(np.atleast_2d(np.asarray(q)), dtype=np.float32)):.1f} us")
print(f"stream_ptr    {t(lambda: js._lib.stream_ptr()):.1f} us")
