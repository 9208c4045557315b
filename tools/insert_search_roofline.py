"""Roofline of the construction's phase-1 search (exact f32 rows from HBM) on one
100K-row streaming batch into N rows (DEEP-shaped 96-d): algorithmic bytes from the
batch's own work counters (hops x (4R + 4) adjacency + evals x (4D + 4) rows+norm +
4D per query), kernel time from CUDA events around a re-run of the same traced
search (the batch's phase 1, on the graph before the batch). Prints one JSON line.
    python tools/insert_search_roofline.py N"""
import importlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_07048_b200 as jb
from paper_2601_07048_b200 import search as js

jbuild = importlib.import_module("paper_2601_07048_b200.build")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_000
nb = 100_000
x = jb.gen_lowrank(n + nb, 96, seed=1, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
p = jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2, max_batch=nb)
g = jb.GraphIndex(capacity=n + nb, degree_cap=32)
jb.insert_stream(g, ds, range(0, n), p)
torch.cuda.synchronize()
# the batch's phase 1 = traced exact search of rows [n, n + nb) on the n-row graph
q = ds.device().x[n:n + nb].contiguous()
bound = js._Bound(ds, q)
cap = 4 * 64 + 64
for _ in range(2):
    fk, hops, evals, flags, tids, _ = js._launch(g, bound, 64, None, cap)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fk, hops, evals, flags, tids, _ = js._launch(g, bound, 64, None, cap)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = float(np.median(ts))
# reference-defined evals (re-evaluations after visited-table evictions excluded)
adj, _ = g.device()
ev = evals.clone()
jb._lib.check(jb._lib.lib().jb_count_evals(jb._lib.ptr(adj), 32, jb._lib.ptr(tids), cap, jb._lib.ptr(hops), None,
                                          g.entry_point, None, nb, jb._lib.ptr(ev), jb._lib.stream_ptr()))
torch.cuda.synchronize()
H, E, Edev = hops.double().sum().item(), ev.double().sum().item(), evals.double().sum().item()
D, R = 96, 32
alg = H * (4 * R + 4) + E * (4 * D + 4) + nb * 4 * D
try:
    peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                              "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    peak = 6650.0
gbs = alg / (ms / 1e3) / 1e9
print(json.dumps({"kernel": "beam_search_kernel<EXACT> (phase-1 traced search of a 100K batch)", "base_rows": n,
                  "queries": nb, "L": 64, "kernel_ms": round(ms, 3), "hops_per_query": round(H / nb, 2),
                  "evals_reference_per_query": round(E / nb, 1), "evals_device_per_query": round(Edev / nb, 1),
                  "alg_bytes": int(alg), "achieved_gbs": round(gbs, 1), "peak_gbs": peak,
                  "frac": round(gbs / peak, 4)}))
