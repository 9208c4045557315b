"""Randomized search parity vs the oracle: exact and bit-exact RaBitQ sources, top-k with
rerank, over random D / R / L / k / bits (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

import paper_2601_07048_b200 as jb
from conftest import gaussian, lowrank
from oracle import rabitq as orq
from oracle import search as osr
from oracle import vamana

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
cases = int(sys.argv[2]) if len(sys.argv) > 2 else 20
bad = 0
for c in range(cases):
    n = int(rng.integers(300, int(os.environ.get("FUZZ_NMAX", "3000"))))
    D = int(rng.choice([int(v) for v in os.environ.get("FUZZ_DIMS", "5,16,33,64,100,128").split(",")]))
    R = int(rng.choice([int(v) for v in os.environ.get("FUZZ_R", "6,16,32,48,64").split(",")]))
    L = int(rng.choice([int(v) for v in os.environ.get("FUZZ_L", "1,7,32,64,200,512").split(",")]))
    k = min(L, int(rng.choice([1, 5, 10, 50])))
    bits = int(rng.choice([1, 2, 4, 8]))
    x = gaussian(n, D, c) if rng.random() < 0.5 else lowrank(n, D, min(D, 8), 0.05, c)
    q = gaussian(64, D, 1000 + c)
    og = vamana.build(x, R=R, L=max(R, 32), alpha=1.2)
    g = jb.GraphIndex(n, R)
    g.adjacency[:n] = og.adj[:n]
    g.degrees[:n] = og.deg[:n]
    g.active_count, g.entry_point = n, og.entry
    ds = jb.VectorDataset(x)
    # exact
    ores = osr.beam_search(og.adj, og.active, og.entry, osr.ExactSource(x, q), len(q), L)
    oi, od = osr.topk(ores, k)
    gi, gd = jb.search_knn_batch(g, ds, q, jb.SearchParams(beam_width=L, k=k))
    ok_e = np.array_equal(gi, oi) and np.array_equal(gd, od)
    # RaBitQ (bit-exact estimator) + rerank
    idx = jb.rabitq_fit(ds, bits=bits, seed=c)
    rot, qadd, sumq = orq.bind(q, idx.centroid, bits, c)
    src = orq.QuantSource(idx.codes, idx.meta, bits, D, rot, qadd, sumq)
    rres = osr.beam_search(og.adj, og.active, og.entry, src, len(q), L)
    ri, rd = osr.topk(rres, k, queries=q, rerank_data=x)
    hi, hd = jb.search_knn_batch(g, idx, q, jb.SearchParams(beam_width=L, k=k, rerank=True), exact_data=ds)
    ok_r = np.array_equal(hi, ri) and np.array_equal(hd, rd)
    bad += (not ok_e) + (not ok_r)
    print(f"case {c}: n={n} D={D} R={R} L={L} k={k} bits={bits}: exact {'OK' if ok_e else 'MISMATCH'}, "
          f"rabitq {'OK' if ok_r else 'MISMATCH'}", flush=True)
print("mismatches", bad)
