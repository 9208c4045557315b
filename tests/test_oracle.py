"""CPU-only: the oracle restatement is pinned to the live reference's outputs
(tests/golden, produced by tests/golden/make_golden.py) and to SPEC.md KATs."""

import numpy as np
import pytest

from conftest import gaussian, golden, lowrank, split, u8_rows
from oracle import knn, rabitq, search, vamana


def _graph_from(f):
    n = int(f["active"])
    g = vamana.Graph(n, f["adjacency"].shape[1])
    g.adj[:] = f["adjacency"]
    g.deg[:] = f["degrees"]
    g.active, g.entry = n, int(f["entry"])
    return g


def _check_results(res, f, prefix):
    fl = split(f[prefix + "frontier_ids"], f[prefix + "frontier_ids_len"])
    fd = split(f[prefix + "frontier_dists"], f[prefix + "frontier_dists_len"])
    vl = split(f[prefix + "visited_ids"], f[prefix + "visited_ids_len"])
    vd = split(f[prefix + "visited_dists"], f[prefix + "visited_dists_len"])
    for i, r in enumerate(res):
        np.testing.assert_array_equal(r.frontier_ids, fl[i])
        np.testing.assert_array_equal(r.frontier_dists, fd[i])
        np.testing.assert_array_equal(r.visited_ids, vl[i])
        np.testing.assert_array_equal(r.visited_dists, vd[i])
        assert r.hops == f[prefix + "hops"][i]
        assert r.evals == f[prefix + "evals"][i]


def test_build_matches_reference_g32():
    f = golden("g32")
    g = vamana.build(gaussian(3000, 32, 0), R=16, L=32, alpha=1.2)
    np.testing.assert_array_equal(g.adj, f["adjacency"])
    np.testing.assert_array_equal(g.deg, f["degrees"])
    assert g.entry == int(f["entry"])


def test_two_pass_build_matches_reference():
    f = golden("two_pass")
    g = vamana.build(gaussian(1500, 32, 21), R=16, L=32, alpha=1.2, max_batch=400, two_pass=True)
    np.testing.assert_array_equal(g.adj, f["adjacency"])
    np.testing.assert_array_equal(g.deg, f["degrees"])
    assert g.entry == int(f["entry"])


def test_build_matches_reference_g33_odd_dims():
    f = golden("g33")
    g = vamana.build(gaussian(800, 33, 5), R=8, L=16, alpha=1.3)
    np.testing.assert_array_equal(g.adj, f["adjacency"])
    assert g.entry == int(f["entry"])


@pytest.mark.parametrize("L", [32, 8])
def test_search_matches_reference_g32(L):
    f = golden("g32")
    x, q = gaussian(3000, 32, 0), gaussian(200, 32, 1)
    g = _graph_from(f)
    res = search.beam_search(g.adj, g.active, g.entry, search.ExactSource(x, q), len(q), L)
    _check_results(res, f, f"L{L}_")


def test_search_matches_reference_g33():
    f = golden("g33")
    x, q = gaussian(800, 33, 5), gaussian(64, 33, 6)
    g = _graph_from(f)
    res = search.beam_search(g.adj, g.active, g.entry, search.ExactSource(x, q), len(q), 16)
    _check_results(res, f, "L16_")


def test_knn_topk_matches_reference():
    f = golden("g32")
    x, q = gaussian(3000, 32, 0), gaussian(200, 32, 1)
    g = _graph_from(f)
    res = search.beam_search(g.adj, g.active, g.entry, search.ExactSource(x, q), len(q), 32)
    ids, ds = search.topk(res, 10)
    np.testing.assert_array_equal(ids, f["knn_ids"])
    np.testing.assert_array_equal(ds, f["knn_dists"])


def test_build_and_stream_match_reference_g128():
    f = golden("g128")
    x = lowrank(4000, 128, 12, 0.05, 7)
    g = vamana.build(x, R=32, L=64, alpha=1.2)
    np.testing.assert_array_equal(g.adj, f["adjacency"])
    q = lowrank(100, 128, 12, 0.05, 8)
    res = search.beam_search(g.adj, g.active, g.entry, search.ExactSource(x, q), len(q), 64)
    _check_results(res, f, "L64_")
    inc = vamana.Graph(4000, 32)
    vamana.batch_insert(inc, x, 0, 33, 32, 64, 1.2)
    vamana.insert_stream(inc, x, 33, 1200, 32, 64, 1.2, max_batch=80)
    np.testing.assert_array_equal(inc.adj[:1200], f["inc_adjacency"])
    assert inc.entry == int(f["inc_entry"])


@pytest.mark.parametrize("bits", [1, 2, 4, 8])
def test_rabitq_fit_bind_match_reference(bits):
    f = golden("rabitq")
    x, qq = gaussian(2000, 128, 2), gaussian(50, 128, 4)
    c, codes, meta = rabitq.fit(x, bits, 3)
    np.testing.assert_array_equal(c, f[f"m{bits}_centroid"])
    np.testing.assert_array_equal(codes, f[f"m{bits}_codes"])
    np.testing.assert_array_equal(meta.view(np.uint32), f[f"m{bits}_meta"].view(np.uint32))
    rot, qadd, sumq = rabitq.bind(qq, c, bits, 3)
    np.testing.assert_array_equal(rot, f[f"m{bits}_rotated"])
    np.testing.assert_array_equal(qadd, f[f"m{bits}_qadd"])
    np.testing.assert_array_equal(sumq, f[f"m{bits}_sumq"])


@pytest.mark.parametrize("bits,tag", [(1, "q1"), (4, "q4")])
def test_rabitq_search_and_rerank_match_reference(bits, tag):
    f, fr = golden("g32"), golden("rabitq")
    x, q = gaussian(3000, 32, 0), gaussian(200, 32, 1)
    g = _graph_from(f)
    c, codes, meta = rabitq.fit(x, bits, 11)
    rot, qadd, sumq = rabitq.bind(q, c, bits, 11)
    src = rabitq.QuantSource(codes, meta, bits, 32, rot, qadd, sumq)
    res = search.beam_search(g.adj, g.active, g.entry, src, len(q), 32)
    _check_results(res, fr, tag + "_")
    ids, ds = search.topk(res, 10, queries=q, rerank_data=x)
    np.testing.assert_array_equal(ids, fr[tag + "_rr_ids"])
    np.testing.assert_array_equal(ds, fr[tag + "_rr_dists"])


def test_exact_knn_and_medoid_match_reference():
    f = golden("misc")
    x, q = gaussian(3000, 32, 0), gaussian(200, 32, 1)
    ids, ds = knn.exact_knn(x, q, 20)
    np.testing.assert_array_equal(ids, f["gt_ids"])
    np.testing.assert_array_equal(ds, f["gt_dists"])
    assert vamana.medoid(x) == int(f["medoid32"])
    assert vamana.medoid(lowrank(4000, 128, 12, 0.05, 7)) == int(f["medoid128"])


# ---- SPEC.md known-answer tests -------------------

def _pts(rows):
    return np.asarray(rows, dtype=np.float32)


def test_prune_kats():
    # line x=1,2 with alpha=1 keeps only x=1
    x = _pts([[0, 0], [1, 0], [2, 0]])
    d = vamana.Pairwise(x)
    kept, _ = vamana.robust_prune(0, [1, 2], d(0, [1, 2]), 1.0, 4, d)
    assert kept.tolist() == [1]
    x = _pts([[0, 0], [1, 0], [0, 3]])
    d = vamana.Pairwise(x)
    kept, _ = vamana.robust_prune(0, [1, 2], d(0, [1, 2]), 1.0, 4, d)
    assert kept.tolist() == [1, 2]
    x = _pts([[0, 0], [1, 0], [0, 1]])
    d = vamana.Pairwise(x)
    kept, _ = vamana.robust_prune(0, [1, 2], d(0, [1, 2]), 1.2, 4, d)
    assert sorted(kept.tolist()) == [1, 2]


def test_path_graph_kat():
    # path graph 0..9 on a line, query at x=9, L=1: visits 0..9, frontier [9]
    x = np.arange(10, dtype=np.float32)[:, None]
    adj = np.full((10, 2), -1, dtype=np.int32)
    for i in range(9):
        adj[i, 0] = i + 1
    res = search.beam_search(adj, 10, 0, search.ExactSource(x, _pts([[9]])), 1, 1)[0]
    assert res.visited_ids.tolist() == list(range(10))
    assert res.frontier_ids.tolist() == [9]


def test_recall_threshold_matching():
    gt_ids = np.array([[0, 1, 2]])
    gt_d = np.array([[1.0, 2.0, 2.0]], dtype=np.float32)
    assert knn.recall_at_k([[0, 2]], gt_ids, gt_d, 2) == 1.0   # tie at the boundary counts
    assert knn.recall_at_k([[5, 0]], gt_ids, gt_d, 2) == 0.5


def test_u8_build_search_knn_match_reference():
    f = golden("u8")
    rows = u8_rows(2600, 32, 31)
    data, q = rows[:2500], rows[2500:]
    g = vamana.build(data, R=16, L=32, alpha=1.2, max_batch=700)
    np.testing.assert_array_equal(g.adj, f["adjacency"])
    np.testing.assert_array_equal(g.deg, f["degrees"])
    assert g.entry == int(f["entry"])
    res = search.beam_search(g.adj, g.active, g.entry, search.ExactSource(data, q), len(q), 32)
    _check_results(res, f, "L32_")
    ids, ds = knn.exact_knn(data, q, 10)
    np.testing.assert_array_equal(ids, f["gt_ids"])
    np.testing.assert_array_equal(ds, f["gt_dists"])
    assert vamana.medoid(data) == int(f["medoid"])
    with pytest.raises(ValueError, match="u8 dataset requires u8 queries"):
        search.ExactSource(data, q.astype(np.float32))


@pytest.mark.parametrize("tag,bits,two", [("m1", 1, False), ("m4", 4, False), ("m4_2p", 4, True)])
def test_quantized_construction_matches_reference(tag, bits, two):
    f = golden("quantized")
    x = gaussian(1200, 32, 51)
    c, codes, meta = rabitq.fit(x, bits, 52)
    g = vamana.build(x, R=16, L=32, alpha=1.2, max_batch=300, two_pass=two,
                     quant=vamana.Quant(c, codes, meta, bits, 52))
    np.testing.assert_array_equal(g.adj, f[tag + "_adjacency"])
    np.testing.assert_array_equal(g.deg, f[tag + "_degrees"])
    assert g.entry == int(f[tag + "_entry"])


def test_mips_augment_and_inner_product_gt_match_reference():
    f = golden("mips")
    data = gaussian(2000, 24, 61) * np.linspace(0.5, 2.0, 2000, dtype=np.float32)[:, None]
    q = gaussian(60, 24, 62)
    ad, aq, m = knn.mips_augment(data, q)
    np.testing.assert_array_equal(ad, f["aug_data"])
    np.testing.assert_array_equal(aq, f["aug_queries"])
    assert m == float(f["max_norm"])
    ids, ds = knn.exact_knn(data, q, 10, inner_product=True)
    np.testing.assert_array_equal(ids, f["gt_ids"])
    np.testing.assert_array_equal(ds, f["gt_dists"])
    g = vamana.build(ad, R=16, L=32, alpha=1.2)
    np.testing.assert_array_equal(g.adj, f["adjacency"])
