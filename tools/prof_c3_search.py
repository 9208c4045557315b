"""Profile target for the C3 (1M x 960, RaBitQ m=4) search kernel (dev tool): one
10K-query batch at L between cudaProfilerStart/Stop.
    python tools/prof_c3_search.py [L] [estimator]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_07048_b200 as jb

L = int(sys.argv[1]) if len(sys.argv) > 1 else 64
est = sys.argv[2] if len(sys.argv) > 2 else "reference"
x = jb.gen_lowrank(1_000_000, 960, seed=1, d_int=16, noise=0.05, basis_seed=0)
q = jb.gen_lowrank(10_000, 960, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
idx = jb.rabitq_fit(ds, bits=4, seed=1)
qd = torch.from_numpy(q).cuda()
sp = jb.SearchParams(beam_width=L, k=10, rerank=True, estimator=est)
for _ in range(2):
    jb.search_knn_batch_device(g, idx, qd, sp, exact_data=ds)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
jb.search_knn_batch_device(g, idx, qd, sp, exact_data=ds)
b.record()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(f"C3 search L={L} {est}: {a.elapsed_time(b):.3f} ms per 10K queries", flush=True)
