"""Host-API (e2e) search with pinned queries (the bench's e2e setup): first-chunk size
sweep (JB_HOST_FIRST), interleaved, vs the device-resident path (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_07048_b200 as jb

x = jb.gen_lowrank(1_000_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
q = jb.gen_lowrank(10_000, 128, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
idx = jb.rabitq_fit(ds, bits=1, seed=1)
qh_t = torch.empty(q.shape, dtype=torch.float32, pin_memory=True)
qh = qh_t.numpy()
qh[...] = q
qd = qh_t.cuda()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
firsts = [int(v) for v in (sys.argv[1:] or ["0", "500", "1000", "2000", "3000"])]
sp = jb.SearchParams(beam_width=128, k=10, rerank=True, estimator="popcount")
ref = None
times = {f: [] for f in firsts}
dev = []
for rep in range(12):
    for f in firsts:
        os.environ["JB_HOST_FIRST"] = str(f)
        flush.fill_(float(rep))
        torch.cuda.synchronize()
        t = time.perf_counter()
        ids, dd = jb.search_knn_batch(g, idx, qh, sp, exact_data=ds)
        times[f].append(time.perf_counter() - t)
        if ref is None:
            ref = ids.copy()
        assert np.array_equal(ids, ref)
    os.environ.pop("JB_HOST_FIRST", None)
    flush.fill_(0.0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    jb.search_knn_batch_device(g, idx, qd, sp, exact_data=ds)
    torch.cuda.synchronize()
    dev.append(time.perf_counter() - t)
for f in firsts:
    tt = times[f][2:]
    print(f"first {f:5d}: median {np.median(tt) * 1e3:.3f} ms min {np.min(tt) * 1e3:.3f} -> {1e4 / np.median(tt) / 1e6:.2f} MQPS")
print(f"device path (wall, incl. sync): median {np.median(dev[2:]) * 1e3:.3f} ms")
