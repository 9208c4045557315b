"""Host-buffer search_knn_batch vs pipeline chunk size (pinned queries), 1M x 128 bench index (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_07048_b200 as jb
from paper_2601_07048_b200 import search as js

x = jb.gen_lowrank(1_000_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
q = jb.gen_lowrank(10_000, 128, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
idx = jb.rabitq_fit(ds, bits=1, seed=1)
qp = torch.empty(q.shape, dtype=torch.float32, pin_memory=True).numpy()
qp[...] = q
sp = jb.SearchParams(beam_width=128, k=10, rerank=True, estimator="popcount")
for chunk in [int(v) for v in sys.argv[1:]] or (0, 3334, 2500, 5000, 10000):
    js.PIPELINE["chunk"] = chunk
    for _ in range(3):
        jb.search_knn_batch(g, idx, qp, sp, exact_data=ds)
    ts = []
    for _ in range(15):
        t = time.perf_counter()
        jb.search_knn_batch(g, idx, qp, sp, exact_data=ds)
        ts.append(time.perf_counter() - t)
    print(f"chunk {chunk:5d}: median {1e3 * np.median(ts):.3f} ms  {10_000 / np.median(ts) / 1e6:.2f} MQPS", flush=True)

# fixed per-call overhead (tiny batch) and the HBM-resident API for comparison
js.PIPELINE["chunk"] = 0
for nq in (32, 10_000):
    qq = qp[:nq]
    for _ in range(3):
        jb.search_knn_batch(g, idx, qq, sp, exact_data=ds)
    ts = []
    for _ in range(15):
        t = time.perf_counter()
        jb.search_knn_batch(g, idx, qq, sp, exact_data=ds)
        ts.append(time.perf_counter() - t)
    print(f"host nq={nq}: median {1e3 * np.median(ts):.3f} ms", flush=True)
qd = torch.from_numpy(q).cuda()
for _ in range(3):
    jb.search_knn_batch_device(g, idx, qd, sp, exact_data=ds)
torch.cuda.synchronize()
ts = []
for _ in range(15):
    t = time.perf_counter()
    jb.search_knn_batch_device(g, idx, qd, sp, exact_data=ds)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t)
print(f"device API nq=10000: median {1e3 * np.median(ts):.3f} ms", flush=True)
os.environ["JB_PIPE_PROFILE"] = "1"
for _ in range(3):
    jb.search_knn_batch(g, idx, qp, sp, exact_data=ds)

# Python-side cost of one call (cProfile over 20 calls)
import cProfile, pstats
os.environ.pop("JB_PIPE_PROFILE", None)
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    jb.search_knn_batch(g, idx, qp, sp, exact_data=ds)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
