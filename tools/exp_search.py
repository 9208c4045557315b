"""Search-kernel experiments on the bench index (dev tool; not part of the product or the bench contract).

    python tools/exp_search.py            # variant x hash-slot sweep, 10K queries, L=128
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2601_07048_b200 as jb
from paper_2601_07048_b200 import search as js

x = jb.gen_lowrank(1_000_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
q = jb.gen_lowrank(10_000, 128, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
idx = jb.rabitq_fit(ds, bits=1, seed=1)
qd = torch.from_numpy(q).cuda()
gi, gd = bench._gt_device(ds.device().x, qd, 100)
gt = jb.measure.GroundTruth(gi.cpu().numpy().astype(np.int64), gd.cpu().numpy().astype(np.float32))


def t_search(L, est, hs=0, reps=7):
    js.TUNING["hash_slots"] = hs
    b = js._Bound(idx, qd, est)
    for _ in range(2):
        js._launch(g, b, L, None, 0)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, e in ev:
        a.record()
        js._launch(g, b, L, None, 0)
        e.record()
    torch.cuda.synchronize()
    sp = jb.SearchParams(beam_width=L, k=10, rerank=True, estimator=est)
    ids, _ = jb.search_knn_batch_device(g, idx, qd, sp, exact_data=ds)
    r = jb.measure.recall_at_k(ids.cpu().numpy(), gt, 10)
    return float(np.median([a.elapsed_time(e) for a, e in ev])), r


for L in [int(v) for v in sys.argv[1:]] or (96, 112, 120, 128):
    for est in ("reference", "popcount"):
        for hs in [int(v) for v in os.environ.get("JB_EXP_HS", "0,512,1024").split(",")]:
            ms, r = t_search(L, est, hs)
            print(f"{est:9s} L={L} hash {hs:5d} {ms:7.3f} ms  {10000 / ms / 1e3:6.2f} MQPS recall {r:.4f}", flush=True)
