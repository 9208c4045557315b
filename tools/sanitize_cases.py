"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case ...]

Cases (each tiny, so the instrumented run finishes in seconds):
  search     exact + RaBitQ (bit-exact and popcount) searches with a 32-slot visited
             table, so every query's table overflows (lossy path, re-evaluations)
  insert     a streaming build in many small batches, so phase 1-3 and the connectivity
             repair (BFS, donor scan, attach) all run; checked against the oracle
  pipeline   search_knn_batch host pipeline (two streams, chunked) + rerank
  protocol   bound distances, robust prune (row and matrix forms), shard pack/merge
  screen     round-2 re-entry: int8 screen records, screened search and phase-2
             prune, closed-row owner pass (checked against the C oracle)
  staged     round-2 paths: exact search with bulk-staged rows (JB_EXACT_DIRECT=0),
             960-d RaBitQ-4 search with bulk-staged records, a repair-heavy build
             (tensor-core donor screen, Gram-screened owner prune, bulk staging)
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def case_search():
    import paper_2601_07048_b200 as jb
    from conftest import gaussian
    from oracle import search as osearch
    from oracle import vamana
    from paper_2601_07048_b200 import search as js

    x, q = gaussian(1500, 32, 0), gaussian(24, 32, 1)
    og = vamana.build(x, R=16, L=32, alpha=1.2)
    g = jb.GraphIndex(og.adj.shape[0], 16)
    g.adjacency, g.degrees = og.adj, og.deg
    g.active_count, g.entry_point = og.active, og.entry
    js.TUNING["hash_slots"] = 32
    res = jb.run_beam_searches(g, jb.VectorDataset(x), q, 64)
    ores = osearch.beam_search(og.adj, og.active, og.entry, osearch.ExactSource(x, q), len(q), 64)
    assert all(np.array_equal(r.frontier_ids, o.frontier_ids) for r, o in zip(res, ores))
    idx = jb.rabitq_fit(jb.VectorDataset(x), bits=1, seed=3)
    for est in ("reference", "popcount"):
        jb.search_knn_batch(g, idx, q, jb.SearchParams(beam_width=64, k=5, rerank=True, estimator=est),
                            exact_data=jb.VectorDataset(x))
    js.TUNING["hash_slots"] = 0
    print("search ok")


def case_insert():
    import paper_2601_07048_b200 as jb
    from conftest import gaussian
    from oracle import vamana

    x = gaussian(1200, 24, 5)
    p = jb.BuildParams(degree_cap=8, build_beam_width=16, alpha=1.2, max_batch=150)
    g = jb.build(jb.VectorDataset(x), p)
    og = vamana.build(x, R=8, L=16, alpha=1.2, max_batch=150)
    assert np.array_equal(g.adjacency, og.adj)
    print("insert ok")


def case_pipeline():
    import paper_2601_07048_b200 as jb
    from conftest import gaussian
    from paper_2601_07048_b200 import search as js

    x, q = gaussian(2000, 48, 2), gaussian(300, 48, 3)
    ds = jb.VectorDataset(x)
    g = jb.build(ds, jb.BuildParams(degree_cap=12, build_beam_width=24))
    idx = jb.rabitq_fit(ds, bits=4, seed=1)
    js.PIPELINE["chunk"] = 64
    jb.search_knn_batch(g, idx, q, jb.SearchParams(beam_width=32, k=10, rerank=True), exact_data=ds)
    jb.search_knn_batch(g, ds, q, jb.SearchParams(beam_width=32, k=10))
    js.PIPELINE["chunk"] = 0
    print("pipeline ok")


def case_protocol():
    import torch

    import paper_2601_07048_b200 as jb
    from conftest import gaussian
    from oracle import vamana
    from paper_2601_07048_b200 import shard
    from paper_2601_07048_b200.search import bind_distance_source

    x, q = gaussian(400, 33, 4), gaussian(10, 33, 5)
    b = bind_distance_source(jb.VectorDataset(x), q)
    b.distances(np.arange(10).repeat(40), np.arange(400))
    idx = jb.rabitq_fit(jb.VectorDataset(x), bits=2, seed=2)
    idx.bind(q).distances(np.arange(10).repeat(40), np.arange(400))
    d = vamana.Pairwise(x)
    cand = np.arange(1, 100)
    jb.robust_prune(0, cand, d(0, cand), alpha=1.2, degree_cap=10, dataset=jb.VectorDataset(x))
    jb.robust_prune(0, cand, d(0, cand), alpha=1.2, degree_cap=10, dist_fn=lambda p, ids: d(p, ids))
    ids = torch.randint(0, 100, (3, 50, 10), dtype=torch.int32, device="cuda").sort(dim=2).values
    dd = torch.rand(3, 50, 10, dtype=torch.float64, device="cuda").sort(dim=2).values
    shard.merge_topk_device(ids, dd, [0, 100, 200], 10)
    rec = torch.stack([shard.pack_topk_device(ids[s], dd[s], 100 * s) for s in range(3)])
    shard.merge_records_device(rec, 10)
    torch.cuda.synchronize()
    print("protocol ok")


def case_staged():
    import paper_2601_07048_b200 as jb
    from conftest import gaussian, lowrank
    from oracle import vamana

    os.environ["JB_EXACT_DIRECT"] = "0"
    x, q = gaussian(3000, 64, 7), gaussian(40, 64, 8)
    p = jb.BuildParams(degree_cap=16, build_beam_width=32, alpha=1.2, max_batch=600)
    g = jb.build(jb.VectorDataset(x), p)
    og = vamana.build(x, R=16, L=32, alpha=1.2, max_batch=600)
    assert np.array_equal(g.adjacency, og.adj)
    jb.search_knn_batch(g, jb.VectorDataset(x), q, jb.SearchParams(beam_width=32, k=10))
    xh, qh = lowrank(600, 960, 16, 0.05, 9), lowrank(8, 960, 16, 0.05, 10)
    dh = jb.VectorDataset(xh)
    gh = jb.build(dh, jb.BuildParams(degree_cap=8, build_beam_width=16, alpha=1.2))
    ih = jb.rabitq_fit(dh, bits=4, seed=3)
    for est in ("reference", "popcount"):
        jb.search_knn_batch(gh, ih, qh, jb.SearchParams(beam_width=16, k=5, rerank=True, estimator=est), exact_data=dh)
    print("staged ok")


def case_screen():
    """round-2 re-entry paths: int8 screen records, screened exact search (16-row
    stage, chain-split A1, next-hop prefetch), screened phase-2 prune, closed-row
    owner pass; D = 40 exercises zero-padded code words."""
    import paper_2601_07048_b200 as jb
    from conftest import gaussian, lowrank
    from oracle import cref
    from paper_2601_07048_b200 import search as js

    os.environ["JB_EXACT_DIRECT"] = "0"
    for x in (lowrank(2500, 64, 12, 0.05, 21), gaussian(2000, 40, 22)):
        p = jb.BuildParams(degree_cap=12, build_beam_width=24, alpha=1.2, max_batch=500)
        g = jb.build(jb.VectorDataset(x), p)
        ref = cref.build(x, 12, 24, 1.2, max_batch=500)
        assert np.array_equal(g.host_adjacency()[: g.active_count], ref.adj[: g.active_count])
        q = x[:30] + 0.01
        res = js.run_beam_searches(g, jb.VectorDataset(x), q, 48)
        os.environ["JB_SEARCH_SCREEN"] = "0"
        res0 = js.run_beam_searches(g, jb.VectorDataset(x), q, 48)
        os.environ.pop("JB_SEARCH_SCREEN")
        assert all(np.array_equal(a.frontier_ids, b.frontier_ids) for a, b in zip(res, res0))
    print("screen ok")


if __name__ == "__main__":
    import torch

    torch.cuda.set_device(0)
    for name in (sys.argv[1:] or ["search", "insert", "pipeline", "protocol", "staged"]):
        globals()["case_" + name]()
