"""Break down the host-buffer search_knn_batch call (e2e path)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_07048_b200 as jb
from paper_2601_07048_b200 import search as js

x = jb.gen_lowrank(1_000_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
q = jb.gen_lowrank(10_000, 128, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
idx = jb.rabitq_fit(ds, bits=1, seed=1)
sp = jb.SearchParams(beam_width=128, k=10, rerank=True, estimator="popcount")
for _ in range(3):
    jb.search_knn_batch(g, idx, q, sp, exact_data=ds)
torch.cuda.synchronize()
T = {}
def tick(name, t0):
    torch.cuda.synchronize(); T[name] = T.get(name, 0) + time.perf_counter() - t0; return time.perf_counter()
for _ in range(10):
    t = time.perf_counter()
    qd = js._queries_to_device(q); t = tick("h2d", t)
    b = js._Bound(idx, qd, "popcount"); t = tick("bind", t)
    fk, *_ = js._launch(g, b, 128, None, 0); t = tick("search", t)
    ids = torch.empty((10000, 10), dtype=torch.int32, device="cuda"); dd = torch.empty((10000, 10), dtype=torch.float64, device="cuda")
    rows = ds.device()
    jb._lib.check(jb._lib.lib().jb_rerank_topk(jb._lib.ptr(rows.x), 128, jb._lib.ptr(qd), 10000, jb._lib.ptr(fk), 128, 10, jb._lib.ptr(ids), jb._lib.ptr(dd), jb._lib.stream_ptr())); t = tick("rerank", t)
    h = js._to_host(ids, dd); t = tick("d2h", t)
print({k: round(v / 10 * 1e3, 3) for k, v in T.items()}, "ms per call")
ts = []
for _ in range(10):
    torch.cuda.synchronize(); t = time.perf_counter()
    jb.search_knn_batch(g, idx, q, sp, exact_data=ds)
    ts.append(time.perf_counter() - t)
print("search_knn_batch e2e", round(np.median(ts) * 1e3, 3), "ms")
