"""Host-API (e2e) search: pipeline chunk sweep vs the device-resident path (dev tool)."""
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
qd = torch.from_numpy(q).cuda()
for est in ("popcount", "reference"):
    sp = jb.SearchParams(beam_width=128, k=10, rerank=True, estimator=est)
    for _ in range(3):
        jb.search_knn_batch_device(g, idx, qd, sp, exact_data=ds)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(20e-3 * 1.9e9))
    a.record()
    for _ in range(10):
        jb.search_knn_batch_device(g, idx, qd, sp, exact_data=ds)
    b.record()
    torch.cuda.synchronize()
    print(f"[{est}] device path {a.elapsed_time(b) / 10:.3f} ms / 10K", flush=True)
    for chunk in (0, 1250, 2500, 3334, 5000, 10000):
        js.PIPELINE["chunk"] = chunk
        for _ in range(3):
            jb.search_knn_batch(g, idx, q, sp, exact_data=ds)
        ts = []
        for _ in range(10):
            t = time.perf_counter()
            jb.search_knn_batch(g, idx, q, sp, exact_data=ds)
            ts.append(time.perf_counter() - t)
        print(f"[{est}] host pipeline chunk {chunk:5d}: median {np.median(ts) * 1e3:.3f} ms "
              f"min {np.min(ts) * 1e3:.3f} ms -> {10000 / np.median(ts) / 1e6:.2f} MQPS", flush=True)
    js.PIPELINE["chunk"] = 0
