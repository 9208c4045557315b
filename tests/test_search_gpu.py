"""GPU parity: the sm_100a search / RaBitQ kernels vs the oracle and the live
reference's golden outputs (identical ids, dists, traces, stats)."""

import numpy as np
import pytest

from conftest import gaussian, golden, lowrank, split, u8_rows
from oracle import knn as oknn
from oracle import rabitq as orabitq
from oracle import search as osearch
from oracle import vamana

pytestmark = pytest.mark.gpu

jb = pytest.importorskip("paper_2601_07048_b200")


def _graph(f):
    n = int(f["active"])
    g = jb.GraphIndex(n, f["adjacency"].shape[1])
    g.adjacency[:] = f["adjacency"]
    g.degrees[:] = f["degrees"]
    g.active_count, g.entry_point = n, int(f["entry"])
    return g


def _graph_from_oracle(og):
    g = jb.GraphIndex(og.adj.shape[0], og.R)
    g.adjacency[:] = og.adj
    g.degrees[:] = og.deg
    g.active_count, g.entry_point = og.active, og.entry
    return g


def _assert_same(res, exp_fids, exp_fd, exp_vids, exp_vd, exp_hops, exp_evals=None):
    for i, r in enumerate(res):
        np.testing.assert_array_equal(r.frontier_ids, exp_fids[i], err_msg=f"query {i} frontier")
        np.testing.assert_array_equal(r.frontier_dists, exp_fd[i], err_msg=f"query {i} frontier dists")
        np.testing.assert_array_equal(r.visited_ids, exp_vids[i], err_msg=f"query {i} trace")
        np.testing.assert_array_equal(r.visited_dists, exp_vd[i], err_msg=f"query {i} trace dists")
        assert r.stats.hops == exp_hops[i], f"query {i} hops"
        if exp_evals is not None:
            assert r.stats.distance_evals == exp_evals[i], f"query {i} evals {r.stats.distance_evals} != {exp_evals[i]}"


def _golden_check(res, f, p):
    _assert_same(res, split(f[p + "frontier_ids"], f[p + "frontier_ids_len"]),
                 split(f[p + "frontier_dists"], f[p + "frontier_dists_len"]),
                 split(f[p + "visited_ids"], f[p + "visited_ids_len"]),
                 split(f[p + "visited_dists"], f[p + "visited_dists_len"]), f[p + "hops"], f[p + "evals"])


def _oracle_check(res, ores, evals=True):
    _assert_same(res, [r.frontier_ids for r in ores], [r.frontier_dists for r in ores],
                 [r.visited_ids for r in ores], [r.visited_dists for r in ores], [r.hops for r in ores],
                 [r.evals for r in ores] if evals else None)


@pytest.mark.parametrize("L", [32, 8])
def test_exact_search_matches_reference_golden(L):
    f = golden("g32")
    x, q = gaussian(3000, 32, 0), gaussian(200, 32, 1)
    res = jb.run_beam_searches(_graph(f), jb.VectorDataset(x), q, L)
    _golden_check(res, f, f"L{L}_")


def test_exact_search_odd_dims_golden():
    f = golden("g33")
    x, q = gaussian(800, 33, 5), gaussian(64, 33, 6)
    _golden_check(jb.run_beam_searches(_graph(f), jb.VectorDataset(x), q, 16), f, "L16_")


def test_exact_search_128d_golden():
    f = golden("g128")
    x, q = lowrank(4000, 128, 12, 0.05, 7), lowrank(100, 128, 12, 0.05, 8)
    _golden_check(jb.run_beam_searches(_graph(f), jb.VectorDataset(x), q, 64), f, "L64_")


def test_knn_batch_matches_reference_golden():
    f = golden("g32")
    x, q = gaussian(3000, 32, 0), gaussian(200, 32, 1)
    ids, ds = jb.search_knn_batch(_graph(f), jb.VectorDataset(x), q, jb.SearchParams(beam_width=32, k=10))
    np.testing.assert_array_equal(ids, f["knn_ids"])
    np.testing.assert_array_equal(ds, f["knn_dists"])
    assert ids.dtype == np.int32 and ds.dtype == np.float64


@pytest.fixture(scope="module")
def graph64():
    x = gaussian(6000, 64, 21)
    og = vamana.build(x, R=24, L=48, alpha=1.2)
    return x, og


@pytest.mark.parametrize("L", [1, 16, 100, 256, 1024])
def test_exact_search_matches_oracle_many_widths(graph64, L):
    x, og = graph64
    q = gaussian(300, 64, 22)
    ores = osearch.beam_search(og.adj, og.active, og.entry, osearch.ExactSource(x, q), len(q), L)
    res = jb.run_beam_searches(_graph_from_oracle(og), jb.VectorDataset(x), q, L)
    _oracle_check(res, ores)


def test_lossy_visited_table_keeps_frontier_and_trace(graph64):
    x, og = graph64
    q = gaussian(200, 64, 23)
    L = 128
    ores = osearch.beam_search(og.adj, og.active, og.entry, osearch.ExactSource(x, q), len(q), L)
    starts = np.arange(len(q)) * 131 % og.active
    ores_s = osearch.beam_search(og.adj, og.active, og.entry, osearch.ExactSource(x, q), len(q), L, starts=starts)
    jb.search.TUNING["hash_slots"] = 64   # far too small: forces re-evaluations
    try:
        res = jb.run_beam_searches(_graph_from_oracle(og), jb.VectorDataset(x), q, L)
        res_s = jb.run_beam_searches(_graph_from_oracle(og), jb.VectorDataset(x), q, L, starts=starts)
    finally:
        jb.search.TUNING["hash_slots"] = 0
    # frontier, trace and even the reference's distance_evals stay exact: evicted
    # queries get their count from |{start} U N(expanded)| (search.py semantics),
    # recounted on device (jb_count_evals)
    _oracle_check(res, ores, evals=True)
    _oracle_check(res_s, ores_s, evals=True)


def test_explicit_starts_and_single_query(graph64):
    x, og = graph64
    q = gaussian(40, 64, 24)
    starts = np.arange(40) * 97 % og.active
    ores = osearch.beam_search(og.adj, og.active, og.entry, osearch.ExactSource(x, q), len(q), 24, starts=starts)
    g = _graph_from_oracle(og)
    _oracle_check(jb.run_beam_searches(g, jb.VectorDataset(x), q, 24, starts=starts), ores)
    one = jb.beam_search(g, jb.VectorDataset(x), q[3], jb.SearchParams(beam_width=24), start=int(starts[3]))
    np.testing.assert_array_equal(one.visited_ids, ores[3].visited_ids)
    cands = jb.search_knn(g, jb.VectorDataset(x), q[5], jb.SearchParams(beam_width=24, k=7))
    o5 = osearch.beam_search(og.adj, og.active, og.entry, osearch.ExactSource(x, q[5:6]), 1, 24)[0]
    assert [c.id for c in cands] == o5.frontier_ids[:7].tolist()
    assert [c.dist for c in cands] == o5.frontier_dists[:7].tolist()


def test_degree_cap_above_warp_width():
    x = gaussian(1500, 16, 31)
    og = vamana.build(x, R=48, L=64, alpha=1.2)
    q = gaussian(100, 16, 32)
    ores = osearch.beam_search(og.adj, og.active, og.entry, osearch.ExactSource(x, q), len(q), 64)
    _oracle_check(jb.run_beam_searches(_graph_from_oracle(og), jb.VectorDataset(x), q, 64), ores)


def test_edge_cases_single_vertex_complete_graph_and_path():
    # single vertex
    g = jb.GraphIndex(1, 4)
    g.active_count = 1
    x = gaussian(1, 8, 1)
    r = jb.run_beam_searches(g, jb.VectorDataset(x), gaussian(3, 8, 2), 4)
    assert all(rr.frontier_ids.tolist() == [0] and rr.stats.hops == 1 for rr in r)
    # complete graph N <= R+1 => exact top-k
    n, R = 9, 8
    x = gaussian(n, 5, 3)
    g = jb.GraphIndex(n, R)
    g.active_count = n
    for u in range(n):
        g.set_neighbors(u, [v for v in range(n) if v != u])
    q = gaussian(20, 5, 4)
    ids, _ = jb.search_knn_batch(g, jb.VectorDataset(x), q, jb.SearchParams(beam_width=4, k=4))
    gt, _ = oknn.exact_knn(x, q, 4)
    np.testing.assert_array_equal(ids, gt)
    # path graph KAT
    x = np.arange(10, dtype=np.float32)[:, None]
    g = jb.GraphIndex(10, 2)
    g.active_count = 10
    for i in range(9):
        g.set_neighbors(i, [i + 1])
    r = jb.beam_search(g, jb.VectorDataset(x), np.array([9.0], np.float32), jb.SearchParams(beam_width=1, k=1))
    assert r.visited_ids.tolist() == list(range(10)) and r.frontier_ids.tolist() == [9]
    # k larger than the reachable set pads with -1 / inf (search.py:368-369)
    g3 = jb.GraphIndex(3, 2)
    g3.active_count = 3
    ids, ds = jb.search_knn_batch(g3, jb.VectorDataset(x[:3]), np.array([[0.5]], np.float32),
                                  jb.SearchParams(beam_width=4, k=4))
    assert ids.tolist() == [[0, -1, -1, -1]] and ds[0, 0] == 0.25 and np.isinf(ds[0, 1:]).all()
    # empty query batch
    ids, ds = jb.search_knn_batch(g, jb.VectorDataset(x), np.zeros((0, 1), np.float32),
                                  jb.SearchParams(beam_width=2, k=2))
    assert ids.shape == (0, 2)


def test_validation_errors_match_reference():
    g = jb.GraphIndex(4, 2)
    x = gaussian(4, 3, 0)
    with pytest.raises(ValueError, match="search on an empty graph"):
        jb.run_beam_searches(g, jb.VectorDataset(x), x, 4)
    g.active_count = 4
    with pytest.raises(ValueError, match="beam_width must be in"):
        jb.run_beam_searches(g, jb.VectorDataset(x), x, 2000)
    with pytest.raises(ValueError, match="start vertex out of range"):
        jb.run_beam_searches(g, jb.VectorDataset(x), x, 4, starts=9)
    with pytest.raises(ValueError, match="k must satisfy"):
        jb.SearchParams(beam_width=4, k=5)


# ---- RaBitQ ------------------------------------------------------------------

@pytest.mark.parametrize("bits", [1, 2, 4, 8])
def test_rabitq_fit_and_bind_bit_exact(bits):
    f = golden("rabitq")
    x, qq = gaussian(2000, 128, 2), gaussian(50, 128, 4)
    idx = jb.rabitq_fit(jb.VectorDataset(x), bits=bits, seed=3)
    np.testing.assert_array_equal(idx.centroid, f[f"m{bits}_centroid"])
    np.testing.assert_array_equal(idx.codes, f[f"m{bits}_codes"])
    np.testing.assert_array_equal(idx.meta.view(np.uint32), f[f"m{bits}_meta"].view(np.uint32))
    b = idx.bind(qq)
    rot, qadd, sumq = b.rotated, b.query_add, b.query_sumq
    np.testing.assert_array_equal(rot, f[f"m{bits}_rotated"])
    np.testing.assert_array_equal(qadd, f[f"m{bits}_qadd"])
    np.testing.assert_array_equal(sumq, f[f"m{bits}_sumq"])


@pytest.mark.parametrize("bits,D", [(1, 96), (4, 960), (2, 37), (8, 20)])
def test_rabitq_fit_bit_exact_vs_oracle_shapes(bits, D):
    x = lowrank(3000 if D < 500 else 1200, D, 16, 0.05, 40 + D)
    x[7] = x.astype(np.float64).mean(axis=0).astype(np.float32)  # near-centroid row
    c, codes, meta = orabitq.fit(x, bits, 5)
    idx = jb.rabitq_fit(jb.VectorDataset(x), bits=bits, seed=5)
    np.testing.assert_array_equal(idx.centroid, c)
    np.testing.assert_array_equal(idx.codes, codes)
    np.testing.assert_array_equal(idx.meta.view(np.uint32), meta.view(np.uint32))


@pytest.mark.parametrize("bits,tag", [(1, "q1"), (4, "q4")])
def test_rabitq_search_and_rerank_match_reference_golden(bits, tag):
    f, fr = golden("g32"), golden("rabitq")
    x, q = gaussian(3000, 32, 0), gaussian(200, 32, 1)
    g = _graph(f)
    idx = jb.rabitq_fit(jb.VectorDataset(x), bits=bits, seed=11)
    _golden_check(jb.run_beam_searches(g, idx, q, 32), fr, tag + "_")
    ids, ds = jb.search_knn_batch(g, idx, q, jb.SearchParams(beam_width=32, k=10, rerank=True),
                                  exact_data=jb.VectorDataset(x))
    np.testing.assert_array_equal(ids, fr[tag + "_rr_ids"])
    np.testing.assert_array_equal(ds, fr[tag + "_rr_dists"])
    with pytest.raises(ValueError, match="requires exact_data"):
        jb.search_knn_batch(g, idx, q, jb.SearchParams(beam_width=32, k=10, rerank=True))


def test_rabitq_search_oracle_960d_m4():
    x = lowrank(1500, 960, 32, 0.05, 50)
    og = vamana.build(x, R=16, L=32, alpha=1.2)
    q = lowrank(60, 960, 32, 0.05, 51)
    c, codes, meta = orabitq.fit(x, 4, 9)
    rot, qadd, sumq = orabitq.bind(q, c, 4, 9)
    src = orabitq.QuantSource(codes, meta, 4, 960, rot, qadd, sumq)
    ores = osearch.beam_search(og.adj, og.active, og.entry, src, len(q), 48)
    idx = jb.rabitq_fit(jb.VectorDataset(x), bits=4, seed=9)
    g = _graph_from_oracle(og)
    _oracle_check(jb.run_beam_searches(g, idx, q, 48), ores)
    ids, ds = jb.search_knn_batch(g, idx, q, jb.SearchParams(beam_width=48, k=10, rerank=True),
                                  exact_data=jb.VectorDataset(x))
    oids, ods = osearch.topk(ores, 10, queries=q, rerank_data=x)
    np.testing.assert_array_equal(ids, oids)
    np.testing.assert_array_equal(ds, ods)


@pytest.mark.parametrize("bits,D", [(4, 96), (4, 88), (2, 192), (2, 180), (8, 48), (1, 384)])
def test_rabitq_search_oracle_64b_records(bits, D):
    """64 B records (code <= 48 B + meta): read whole by two 256-bit loads and
    estimated from registers, incl. a partial last code piece (D = 88, 180)."""
    assert jb._lib.lib().jb_rabitq_record_bytes(D, bits) == 64
    x = lowrank(2000, D, 16, 0.05, 60 + D)
    og = vamana.build(x, R=16, L=32, alpha=1.2)
    q = lowrank(80, D, 16, 0.05, 61 + D)
    c, codes, meta = orabitq.fit(x, bits, 5)
    rot, qadd, sumq = orabitq.bind(q, c, bits, 5)
    src = orabitq.QuantSource(codes, meta, bits, D, rot, qadd, sumq)
    ores = osearch.beam_search(og.adj, og.active, og.entry, src, len(q), 40)
    idx = jb.rabitq_fit(jb.VectorDataset(x), bits=bits, seed=5)
    g = _graph_from_oracle(og)
    _oracle_check(jb.run_beam_searches(g, idx, q, 40), ores)


def test_medoid_matches_reference_golden():
    f = golden("misc")
    assert jb.medoid(jb.VectorDataset(gaussian(3000, 32, 0))) == int(f["medoid32"])
    assert jb.medoid(jb.VectorDataset(lowrank(4000, 128, 12, 0.05, 7))) == int(f["medoid128"])


def test_popcount_estimator_recall_tracks_reference_estimator():
    x = jb.gen_lowrank(20000, 128, seed=1, basis_seed=0)
    q = jb.gen_lowrank(300, 128, seed=2, basis_seed=0)
    ds = jb.VectorDataset(x)
    g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
    idx = jb.rabitq_fit(ds, bits=1, seed=1)
    gt_i, gt_d = oknn.exact_knn(x, q, 50)
    gt = jb.GroundTruth(gt_i, gt_d)
    for L in (32, 64):
        r = {}
        for est in ("reference", "popcount"):
            ids, ds_ = jb.search_knn_batch(g, idx, q, jb.SearchParams(beam_width=L, k=10, rerank=True, estimator=est),
                                           exact_data=ds)
            assert np.all(np.diff(ds_, axis=1) >= 0)  # reranked: ascending exact distances
            r[est] = jb.recall_at_k(ids, gt, 10)
        assert r["popcount"] >= r["reference"] - 0.02, r
    # multi-bit codes: the estimator runs over the code bit-planes
    for bits in (2, 4, 8):
        idxm = jb.rabitq_fit(ds, bits=bits, seed=1)
        r = {}
        for est in ("reference", "popcount"):
            ids, _ = jb.search_knn_batch(g, idxm, q, jb.SearchParams(beam_width=48, k=10, rerank=True, estimator=est),
                                         exact_data=ds)
            r[est] = jb.recall_at_k(ids, gt, 10)
        assert r["popcount"] >= r["reference"] - 0.02, (bits, r)


@pytest.mark.parametrize("bits,D", [(2, 100), (4, 960), (8, 20), (1, 64)])
def test_plane_records_match_host_layout(bits, D):
    """jb_rabitq_pack_planes: plane b' bit e = bit b' of the code of dimension e, then meta."""
    x = gaussian(300, D, 8)
    idx = jb.rabitq_fit(jb.VectorDataset(x), bits=bits, seed=4)
    rec, rb = idx.device_planes()
    rec = rec.cpu().numpy()
    pw = ((D + 31) // 32 + 3) & ~3
    u = jb.rabitq.unpack_codes(idx.codes, bits, D).astype(np.uint64)
    for v in (0, 7, 299):
        words = rec[v, : bits * pw * 4].view(np.uint32).reshape(bits, pw)
        for bp in range(bits):
            want = np.zeros(pw, np.uint64)
            for e in range(D):
                want[e // 32] |= ((u[v, e] >> np.uint64(bp)) & np.uint64(1)) << np.uint64(e % 32)
            np.testing.assert_array_equal(words[bp], want.astype(np.uint32))
        np.testing.assert_array_equal(rec[v, bits * pw * 4: bits * pw * 4 + 8].view(np.float32), idx.meta[v])


@pytest.mark.parametrize("chunk", [0, 97, 1000])
@pytest.mark.parametrize("kind", ["exact", "rabitq", "popcount"])
def test_host_pipeline_matches_device_path(chunk, kind):
    """jb_search_knn_host (host buffers, chunked over two streams) returns exactly
    what the HBM-resident path returns, for every chunking."""
    from paper_2601_07048_b200 import search as js

    x = lowrank(6000, 64, 8, 0.05, 21)
    q = lowrank(1000, 64, 8, 0.05, 22)
    ds = jb.VectorDataset(x)
    g = jb.build(ds, jb.BuildParams(degree_cap=24, build_beam_width=48, alpha=1.2))
    if kind == "exact":
        src, sp = ds, jb.SearchParams(beam_width=40, k=10)
    else:
        src = jb.rabitq_fit(ds, bits=1, seed=3)
        sp = jb.SearchParams(beam_width=40, k=10, rerank=True,
                             estimator="popcount" if kind == "popcount" else "reference")
    import torch

    di, dd = jb.search_knn_batch_device(g, src, torch.from_numpy(q).cuda(), sp, exact_data=ds)
    js.PIPELINE["chunk"] = chunk
    try:
        hi, hd = jb.search_knn_batch(g, src, q, sp, exact_data=ds)
        hi2, hd2 = jb.search_knn_batch(g, src, q[:333], sp, exact_data=ds)  # reuse of the cached context
        qp = torch.empty(q.shape, dtype=torch.float32, pin_memory=True).numpy()  # pinned: no staging copy
        qp[...] = q
        hi3, hd3 = jb.search_knn_batch(g, src, qp, sp, exact_data=ds)
        # pageable result arrays through the C ABI: the staged copy-out path
        from paper_2601_07048_b200 import _lib

        plan = js._knn_plan(g, src, q.shape[1], sp, ds)
        hi4 = np.empty((len(q), sp.k), np.int32)
        hd4 = np.empty((len(q), sp.k), np.float64)
        _lib.check(_lib.lib().jb_search_knn_host(_lib.C.byref(plan), _lib.ptr(q), len(q), _lib.ptr(hi4),
                                                 _lib.ptr(hd4), _lib.stream_ptr()))
    finally:
        js.PIPELINE["chunk"] = 0
    np.testing.assert_array_equal(hi, di.cpu().numpy())
    np.testing.assert_array_equal(hd, dd.cpu().numpy())
    np.testing.assert_array_equal(hi2, hi[:333])
    np.testing.assert_array_equal(hd2, hd[:333])
    np.testing.assert_array_equal(hi3, hi)
    np.testing.assert_array_equal(hd3, hd)
    np.testing.assert_array_equal(hi4, hi)
    np.testing.assert_array_equal(hd4, hd)


def test_u8_search_knn_gt_medoid_match_reference_golden():
    f = golden("u8")
    rows = u8_rows(2600, 32, 31)
    data, q = rows[:2500], rows[2500:]
    g, ds = _graph(f), jb.VectorDataset(data)
    _golden_check(jb.run_beam_searches(g, ds, q, 32), f, "L32_")
    ids, dists = jb.search_knn_batch(g, ds, q, jb.SearchParams(beam_width=32, k=10))
    np.testing.assert_array_equal(ids, f["knn_ids"])
    np.testing.assert_array_equal(dists, f["knn_dists"])
    gt = jb.exact_knn(ds, jb.VectorDataset(q), 10)
    np.testing.assert_array_equal(gt.ids, f["gt_ids"])
    np.testing.assert_array_equal(gt.distances, f["gt_dists"])
    assert jb.medoid(ds) == int(f["medoid"])
    with pytest.raises(ValueError, match="u8 dataset requires u8 queries"):
        jb.run_beam_searches(g, ds, q.astype(np.float32), 32)


@pytest.mark.parametrize("L", [8, 64, 300])
def test_u8_search_matches_oracle_128d(L):
    # BigANN shape (128-d u8): 16 B-aligned rows, several beam widths incl. the smem merge path
    rows = u8_rows(3100, 128, 41)
    data, q = rows[:3000], rows[3000:]
    og = vamana.build(data, R=24, L=48, alpha=1.2, max_batch=1000)
    g = _graph_from_oracle(og)
    res = jb.run_beam_searches(g, jb.VectorDataset(data), q, L)
    _oracle_check(res, osearch.beam_search(og.adj, og.active, og.entry, osearch.ExactSource(data, q), len(q), L))


def test_run_queries_threads_and_sweep_match_single_batch():
    """run_queries(workers=N) splits the batch over threads like bench.py:69-91; the
    concurrent native calls (per-thread contexts) return exactly the one-batch result."""
    x = lowrank(4000, 64, 8, 0.05, 81)
    q = lowrank(600, 64, 8, 0.05, 82)
    ds = jb.VectorDataset(x)
    g = jb.build(ds, jb.BuildParams(degree_cap=20, build_beam_width=40, alpha=1.2))
    idx = jb.rabitq_fit(ds, bits=1, seed=7)
    sp = jb.SearchParams(beam_width=40, k=10, rerank=True)
    one = jb.run_queries(g, idx, q, sp, exact_data=ds, workers=1)
    many = jb.run_queries(g, idx, q, sp, exact_data=ds, workers=6)
    np.testing.assert_array_equal(one[0], many[0])
    np.testing.assert_array_equal(one[1], many[1])
    gt = jb.exact_knn(ds, jb.VectorDataset(q), 20)
    pts = jb.sweep(g, ds, q, gt, 10, [16, 32], workers=3)
    assert [p.beam_width for p in pts] == [16, 32] and pts[1].recall >= pts[0].recall > 0.5


def test_search_properties_spec():
    """no double evaluation, deterministic visitation order, recall
    non-decreasing in L."""
    x = lowrank(5000, 48, 8, 0.05, 91)
    q = lowrank(300, 48, 8, 0.05, 92)
    ds = jb.VectorDataset(x)
    g = jb.build(ds, jb.BuildParams(degree_cap=16, build_beam_width=32, alpha=1.2))
    a = jb.run_beam_searches(g, ds, q, 64)
    b = jb.run_beam_searches(g, ds, q, 64)
    for ra, rb in zip(a, b):
        np.testing.assert_array_equal(ra.visited_ids, rb.visited_ids)
        np.testing.assert_array_equal(ra.frontier_ids, rb.frontier_ids)
        assert np.unique(ra.visited_ids).size == ra.visited_ids.size  # every vertex expanded at most once
        # every evaluated id is the start or a neighbour of an expanded vertex, each counted once
        nb = g.adjacency[ra.visited_ids].ravel()
        assert ra.stats.distance_evals == np.unique(np.append(nb[nb >= 0], g.entry_point)).size
    gt = jb.exact_knn(ds, jb.VectorDataset(q), 10)
    rec = [jb.recall_at_k(jb.search_knn_batch(g, ds, q, jb.SearchParams(beam_width=L, k=10))[0], gt, 10)
           for L in (16, 32, 64, 128)]
    assert all(r2 >= r1 - 1e-9 for r1, r2 in zip(rec, rec[1:])), rec


def test_bench_scale_rabitq_fit_and_bind_identical_to_reference():
    """The headline index's RaBitQ codes / metadata / centroid (1M x 128, m=1) and its
    10K bound queries are bit-identical to beamann's (hashes of the reference run)."""
    import hashlib
    import json
    import os

    from conftest import GOLDEN

    ref = json.load(open(os.path.join(GOLDEN, "bench_rabitq.json")))
    h = lambda a: hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    x = jb.gen_lowrank(1_000_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
    q = jb.gen_lowrank(10_000, 128, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
    idx = jb.rabitq_fit(jb.VectorDataset(x), bits=1, seed=1)
    assert h(idx.centroid) == ref["centroid"]
    assert h(idx.codes) == ref["codes"]
    assert h(idx.meta) == ref["meta"]
    b = idx.bind(q)
    rot, qa, qs = b.rotated, b.query_add, b.query_sumq
    assert (h(rot), h(qa), h(qs)) == (ref["rotated"], ref["qadd"], ref["sumq"])


def test_default_params_r64_build_and_search_match_oracle():
    """beamann's defaults (R=64, L=128): the build is identical to the oracle's and
    the two-chunk (R > 32) hop of the search kernel gives identical frontiers."""
    x = lowrank(3000, 24, 8, 0.05, 99)
    q = lowrank(150, 24, 8, 0.05, 98)
    og = vamana.build(x, R=64, L=128, alpha=1.2, max_batch=100_000)
    g = jb.build(jb.VectorDataset(x), jb.BuildParams())
    assert g.entry_point == og.entry
    np.testing.assert_array_equal(g.degrees[:3000], og.deg[:3000])
    np.testing.assert_array_equal(g.adjacency[:3000], og.adj[:3000])
    ores = osearch.beam_search(og.adj, og.active, og.entry, osearch.ExactSource(x, q), len(q), 128)
    _oracle_check(jb.run_beam_searches(g, jb.VectorDataset(x), q, 128), ores)
