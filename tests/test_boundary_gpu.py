"""GPU: the drop-in surface around the kernels — the reference's distance-source
protocol (bind_distance_source / RaBitQIndex.bind -> distances/pack/decode,
search.py:82-168, rabitq.py:170-254), robust_prune with reference-style dist_fn
objects (graph.py:174-228, build.py:105-134), graph slab transfer accounting,
adopted beamann-style graphs, and the argument checks that keep the kernels
in bounds."""

import types

import numpy as np
import pytest

from conftest import gaussian, lowrank, u8_rows
from oracle import cref, rabitq as orq, search as osearch, vamana

pytestmark = pytest.mark.gpu


def test_bound_exact_distances_pack_decode_match_reference():
    import paper_2601_07048_b200 as jb
    from paper_2601_07048_b200.search import ExactDistances, bind_distance_source

    x, q = gaussian(500, 33, 1), gaussian(20, 33, 2)
    ref = osearch.ExactSource(x, q)
    rng = np.random.default_rng(3)
    qr, ids = rng.integers(0, 20, 400), rng.integers(0, 500, 400)
    for b in (bind_distance_source(jb.VectorDataset(x), q), ExactDistances(jb.VectorDataset(x)).bind(q)):
        d = b.distances(qr, ids)
        assert d.dtype == np.float32
        np.testing.assert_array_equal(d, ref(qr, ids))
        keys = b.pack(d, ids)
        np.testing.assert_array_equal(keys, osearch.pack(d, ids))
        np.testing.assert_array_equal(b.decode(keys), osearch.unpack_dist(keys))
        assert b.n_queries == 20
    with pytest.raises(IndexError):
        b.distances([0], [500])
    with pytest.raises(ValueError, match="query dims"):
        bind_distance_source(jb.VectorDataset(x), gaussian(2, 32, 0))
    with pytest.raises(TypeError):
        bind_distance_source(object(), q)


def test_bound_u8_distances_are_exact_integers():
    import paper_2601_07048_b200 as jb
    from paper_2601_07048_b200.search import bind_distance_source

    rows = u8_rows(600, 40, 5)
    data, q = rows[:500], rows[500:]
    b = bind_distance_source(jb.VectorDataset(data), q)
    rng = np.random.default_rng(1)
    qr, ids = rng.integers(0, 100, 300), rng.integers(0, 500, 300)
    d = b.distances(qr, ids)
    np.testing.assert_array_equal(d, osearch.ExactSource(data, q)(qr, ids))
    with pytest.raises(ValueError, match="u8 dataset requires u8 queries"):
        bind_distance_source(jb.VectorDataset(data), q.astype(np.float32))


@pytest.mark.parametrize("bits", [1, 2, 4, 8])
def test_rabitq_bind_returns_reference_bound_estimator(bits):
    import paper_2601_07048_b200 as jb

    x, q = gaussian(800, 48, 3), gaussian(30, 48, 4)
    idx = jb.rabitq_fit(jb.VectorDataset(x), bits=bits, seed=5)
    c, codes, meta = orq.fit(x, bits, 5)
    rot, qadd, sumq = orq.bind(q, c, bits, 5)
    b = idx.bind(q)
    np.testing.assert_array_equal(b.rotated, rot)
    np.testing.assert_array_equal(b.query_add, qadd)
    np.testing.assert_array_equal(b.query_sumq, sumq)
    rng = np.random.default_rng(bits)
    qr, ids = rng.integers(0, 30, 500), rng.integers(0, 800, 500)
    ref = orq.QuantSource(codes, meta, bits, 48, rot, qadd, sumq)
    np.testing.assert_array_equal(b.distances(qr, ids), ref(qr, ids))
    keys = b.pack(b.distances(qr, ids), ids)
    np.testing.assert_array_equal(b.decode(keys), osearch.unpack_dist(keys))


def test_robust_prune_accepts_reference_dist_fns():
    import paper_2601_07048_b200 as jb

    x = lowrank(400, 24, 6, 0.1, 9)
    d = vamana.Pairwise(x)
    rng = np.random.default_rng(0)
    for trial in range(6):
        p = int(rng.integers(0, 400))
        cand = rng.choice(np.delete(np.arange(400), p), size=int(rng.integers(5, 120)), replace=False)
        cd = d(p, cand)
        R, alpha = int(rng.integers(2, 20)), float(rng.choice([1.0, 1.2, 1.5]))
        ok, okd = vamana.robust_prune(p, cand, cd, alpha, R, d)
        # 1. an opaque callable (the oracle's own pairwise): matrix path
        opaque = lambda piv, ids: d(piv, ids)  # noqa: E731
        gk, gkd = jb.robust_prune(p, cand, cd, alpha=alpha, degree_cap=R, dist_fn=opaque)
        np.testing.assert_array_equal(gk, ok)
        np.testing.assert_array_equal(gkd, okd)
        # 2. a beamann-style _PairwiseDistances (rows in `_x`): device pair distances
        ref_like = types.SimpleNamespace(_x=x, _norms=None, _quantizer=None)
        gk, gkd = jb.robust_prune(p, cand, cd, alpha=alpha, degree_cap=R, dist_fn=ref_like)
        np.testing.assert_array_equal(gk, ok)
        # 3. dataset=
        gk, _ = jb.robust_prune(p, cand, cd, alpha=alpha, degree_cap=R, dataset=jb.VectorDataset(x))
        np.testing.assert_array_equal(gk, ok)


def test_robust_prune_u8_and_quantized_sources():
    import paper_2601_07048_b200 as jb

    rows = u8_rows(300, 16, 3)
    d = vamana.Pairwise(rows)
    cand = np.arange(1, 120)
    ok, okd = vamana.robust_prune(0, cand, d(0, cand), 1.2, 10, d)
    gk, gkd = jb.robust_prune(0, cand, d(0, cand), alpha=1.2, degree_cap=10, dataset=jb.VectorDataset(rows))
    np.testing.assert_array_equal(gk, ok)
    np.testing.assert_array_equal(gkd, okd)
    x = gaussian(300, 32, 7)
    c, codes, meta = orq.fit(x, 4, 8)
    qp = vamana.Quant(c, codes, meta, 4, 8).pairwise(x)
    cd = qp(5, cand[cand != 5])
    ok, _ = vamana.robust_prune(5, cand[cand != 5], cd, 1.2, 12, qp)
    idx = jb.rabitq_fit(jb.VectorDataset(x), bits=4, seed=8)
    fn = types.SimpleNamespace(dataset=jb.VectorDataset(x), quantizer=idx)
    gk, _ = jb.robust_prune(5, cand[cand != 5], cd, alpha=1.2, degree_cap=12, dist_fn=fn)
    np.testing.assert_array_equal(gk, ok)


def test_adjacency_reads_do_not_reupload_the_slab():
    import paper_2601_07048_b200 as jb

    x, q = gaussian(3000, 32, 0), gaussian(50, 32, 1)
    ds = jb.VectorDataset(x)
    g = jb.build(ds, jb.BuildParams(degree_cap=16, build_beam_width=32))
    jb.search_knn_batch(g, ds, q, jb.SearchParams(beam_width=32))
    up = g.h2d_bytes
    a, dg = g.adjacency, g.degrees            # downloads once
    _ = a[5, :3].tolist(), int(dg.sum()), (a >= 0).sum()
    r1 = jb.run_beam_searches(g, ds, q, 32)  # read-only use: no upload
    jb.search_knn_batch(g, ds, q, jb.SearchParams(beam_width=32))
    assert g.h2d_bytes == up
    # a write through the tracked view is uploaded before the next device use
    row = g.adjacency[0]
    keep = row[: g.degree(0)].copy()
    row[: keep.size] = keep[::-1]
    jb.run_beam_searches(g, ds, q, 32)
    assert g.h2d_bytes > up
    assert len(r1) == 50


def test_insert_stream_into_adopted_reference_graph_writes_back():
    import paper_2601_07048_b200 as jb

    x = gaussian(1500, 24, 11)
    params = jb.BuildParams(degree_cap=12, build_beam_width=24, alpha=1.2, max_batch=200)
    og = vamana.Graph(1500, 12)
    vamana.batch_insert(og, x, 0, 13, 12, 24, 1.2)
    beam_like = types.SimpleNamespace(adjacency=og.adj.copy(), degrees=og.deg.copy(), entry_point=og.entry,
                                      active_count=og.active, degree_cap=12)
    jb.insert_stream(beam_like, jb.VectorDataset(x), range(13, 900), params)
    vamana.insert_stream(og, x, 13, 900, 12, 24, 1.2, max_batch=200)
    assert beam_like.active_count == 900
    assert beam_like.entry_point == og.entry
    np.testing.assert_array_equal(beam_like.adjacency, og.adj)
    np.testing.assert_array_equal(beam_like.degrees, og.deg)


def test_short_sources_and_u8_rerank():
    import paper_2601_07048_b200 as jb

    x = gaussian(1000, 32, 2)
    ds = jb.VectorDataset(x)
    g = jb.build(ds, jb.BuildParams(degree_cap=12, build_beam_width=24))
    with pytest.raises(ValueError, match="holds 500 vectors"):
        jb.search_knn_batch(g, jb.VectorDataset(x[:500]), x[:3], jb.SearchParams(beam_width=24))
    idx = jb.rabitq_fit(ds, bits=1, seed=1)
    with pytest.raises(ValueError, match="exact_data holds"):
        jb.search_knn_batch(g, idx, x[:3], jb.SearchParams(beam_width=24, rerank=True),
                            exact_data=jb.VectorDataset(x[:10]))
    with pytest.raises(ValueError, match="degree_cap must be <= 128"):
        jb.BuildParams(degree_cap=150)
    # u8 rows as rerank data: widened exactly, as the reference's data[ids].astype(f32)
    rows = u8_rows(1300, 32, 4)
    data, q = rows[:1200], rows[1200:]
    f = data.astype(np.float32)
    gf = jb.build(jb.VectorDataset(f), jb.BuildParams(degree_cap=12, build_beam_width=24))
    qi = jb.rabitq_fit(jb.VectorDataset(f), bits=4, seed=2)
    sp = jb.SearchParams(beam_width=24, k=5, rerank=True)
    ids_u8, d_u8 = jb.search_knn_batch(gf, qi, q.astype(np.float32), sp, exact_data=jb.VectorDataset(data))
    ids_f, d_f = jb.search_knn_batch(gf, qi, q.astype(np.float32), sp, exact_data=jb.VectorDataset(f))
    np.testing.assert_array_equal(ids_u8, ids_f)
    np.testing.assert_array_equal(d_u8, d_f)


def test_large_seed_batch_is_tiled_and_exact():
    """A first batch large enough that the seed prune runs in pivot tiles (scratch bound)
    matches the C oracle's all-pairs seed batch."""
    import paper_2601_07048_b200 as jb

    n = 12_000
    x = lowrank(n, 8, 4, 0.2, 3)
    g = jb.GraphIndex(n, 8)
    jb.batch_insert(g, jb.VectorDataset(x), range(0, n), jb.BuildParams(degree_cap=8, build_beam_width=16))
    og = cref.Graph(n, 8)
    cref.batch_insert(og, cref.Rows(x), 0, n, 16, 1.2)
    np.testing.assert_array_equal(g.adjacency, og.adj)
    assert g.entry_point == og.entry
