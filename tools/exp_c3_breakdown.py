"""960-d (C3-shaped) step breakdown: bind / search / rerank kernel times (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_07048_b200 as jb
from paper_2601_07048_b200 import _lib
from paper_2601_07048_b200 import search as js

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
x = jb.gen_lowrank(n, 960, seed=1, d_int=16, noise=0.05, basis_seed=0)
q = jb.gen_lowrank(10_000, 960, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
idx = jb.rabitq_fit(ds, bits=4, seed=1)
qd = torch.from_numpy(q).cuda()
rows = ds.device()


def ev_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return float(np.median(out))


for est in ("reference", "popcount"):
    tb = ev_time(lambda: js._Bound(idx, qd, est))
    bnd = js._Bound(idx, qd, est)
    ts = ev_time(lambda: js._launch(g, bnd, 64, None, 0))
    fk, *_ = js._launch(g, bnd, 64, None, 0)
    oi = torch.empty((10_000, 10), dtype=torch.int32, device="cuda")
    od = torch.empty((10_000, 10), dtype=torch.float64, device="cuda")
    tr = ev_time(lambda: _lib.check(_lib.lib().jb_rerank_topk(_lib.ptr(rows.x), 960, _lib.ptr(qd), 10_000, _lib.ptr(fk),
                                                              64, 10, _lib.ptr(oi), _lib.ptr(od), _lib.stream_ptr())))
    sp = jb.SearchParams(beam_width=64, k=10, rerank=True, estimator=est)
    tt = ev_time(lambda: jb.search_knn_batch_device(g, idx, qd, sp, exact_data=ds))
    print(f"{est}: bind {tb:.3f} ms, search {ts:.3f} ms, rerank {tr:.3f} ms, device step {tt:.3f} ms", flush=True)
