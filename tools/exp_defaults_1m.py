"""beamann's default parameters at 1M x 128 (BuildParams(): R=64, L=128): build rate and
search QPS / recall (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2601_07048_b200 as jb

x = jb.gen_lowrank(1_000_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
q = jb.gen_lowrank(10_000, 128, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
p = jb.BuildParams()
jb.build(jb.VectorDataset(x[:250_000]), p)
torch.cuda.synchronize()
t = time.perf_counter()
g = jb.build(ds, p)
torch.cuda.synchronize()
tb = time.perf_counter() - t
print(f"default BuildParams (R={p.degree_cap}, L={p.build_beam_width}) 1M x 128: {tb:.2f} s, {1e6 / tb:.0f} inserts/s", flush=True)
qd = torch.from_numpy(q).cuda()
gi, gd = bench._gt_device(ds.device().x, qd, 100)
gt = jb.GroundTruth(gi.cpu().numpy(), gd.cpu().numpy().astype(np.float32))
idx = jb.rabitq_fit(ds, bits=1, seed=1)
for L in (32, 64, 128):
    for name, src, sp in (("exact", ds, jb.SearchParams(beam_width=L, k=10)),
                          ("rabitq1-popcount", idx, jb.SearchParams(beam_width=L, k=10, rerank=True, estimator="popcount"))):
        for _ in range(2):
            jb.search_knn_batch_device(g, src, qd, sp, exact_data=ds)
        torch.cuda.synchronize()
        t = time.perf_counter()
        ids, _ = jb.search_knn_batch_device(g, src, qd, sp, exact_data=ds)
        torch.cuda.synchronize()
        el = time.perf_counter() - t
        r = jb.recall_at_k(ids.cpu().numpy(), gt, 10)
        print(f"  {name} L={L}: {10_000 / el / 1e6:.2f}M QPS, recall@10 {r:.4f}", flush=True)
