"""CPU-only: the C restatement of the oracle (oracle/c/jbo.c via oracle/cref.py)
is pinned to the live reference's fixtures (tests/golden) and to the numpy
oracle. bench.py's CPU legs build and search the 1M workload with it, so its
parity is what makes the reference arm the reference's algorithm."""

import numpy as np
import pytest

from conftest import gaussian, golden, lowrank, split
from oracle import cref, knn, rabitq, search, vamana


def _frontiers_match(keys, hops, evals, f, prefix):
    fl = split(f[prefix + "frontier_ids"], f[prefix + "frontier_ids_len"])
    fd = split(f[prefix + "frontier_dists"], f[prefix + "frontier_dists_len"])
    for i, r in enumerate(cref.results(keys, hops, evals)):
        np.testing.assert_array_equal(r.frontier_ids, fl[i])
        np.testing.assert_array_equal(r.frontier_dists, fd[i])
        assert r.hops == f[prefix + "hops"][i]
        assert r.evals == f[prefix + "evals"][i]


@pytest.mark.parametrize("threads", [1, 4])
def test_c_build_matches_reference_g32(threads):
    f = golden("g32")
    g = cref.build(gaussian(3000, 32, 0), R=16, L=32, alpha=1.2, threads=threads)
    np.testing.assert_array_equal(g.adj, f["adjacency"])
    np.testing.assert_array_equal(g.deg, f["degrees"])
    assert g.entry == int(f["entry"])


def test_c_build_matches_reference_g33_odd_dims():
    f = golden("g33")
    g = cref.build(gaussian(800, 33, 5), R=8, L=16, alpha=1.3)
    np.testing.assert_array_equal(g.adj, f["adjacency"])
    assert g.entry == int(f["entry"])


def test_c_build_stream_and_search_match_reference_g128():
    f = golden("g128")
    x = lowrank(4000, 128, 12, 0.05, 7)
    g = cref.build(x, R=32, L=64, alpha=1.2)
    np.testing.assert_array_equal(g.adj, f["adjacency"])
    rows = cref.Rows(x)
    q = lowrank(100, 128, 12, 0.05, 8)
    _frontiers_match(*cref.search_exact(g.adj, g.active, g.entry, rows, q, 64), f, "L64_")
    inc = cref.Graph(4000, 32)
    cref.batch_insert(inc, rows, 0, 33, 64, 1.2)
    cref.insert_stream(inc, rows, 33, 1200, 64, 1.2, max_batch=80)
    np.testing.assert_array_equal(inc.adj[:1200], f["inc_adjacency"])
    assert inc.entry == int(f["inc_entry"])


@pytest.mark.parametrize("L", [32, 8])
def test_c_search_and_topk_match_reference_g32(L):
    f = golden("g32")
    x, q = gaussian(3000, 32, 0), gaussian(200, 32, 1)
    rows = cref.Rows(x)
    keys, hops, evals = cref.search_exact(f["adjacency"], int(f["active"]), int(f["entry"]), rows, q, L)
    _frontiers_match(keys, hops, evals, f, f"L{L}_")
    if L == 32:
        ids = cref.frontier_ids(keys)
        # search_knn_batch without rerank takes the frontier head; with rerank the C top-k
        np.testing.assert_array_equal(np.where(ids[:, :10] >= 0, ids[:, :10], -1), f["knn_ids"])


@pytest.mark.parametrize("bits,tag", [(1, "q1"), (4, "q4")])
def test_c_rabitq_search_and_rerank_match_reference(bits, tag):
    f, fr = golden("g32"), golden("rabitq")
    x, q = gaussian(3000, 32, 0), gaussian(200, 32, 1)
    quant = cref.Quantized.fit(x, bits, 11)
    keys, hops, evals = cref.search_rabitq(f["adjacency"], int(f["active"]), int(f["entry"]), quant, q, 32)
    _frontiers_match(keys, hops, evals, fr, tag + "_")
    ids, ds = cref.rerank_topk(x, q, cref.frontier_ids(keys), 10)
    np.testing.assert_array_equal(ids, fr[tag + "_rr_ids"])
    np.testing.assert_array_equal(ds, fr[tag + "_rr_dists"])


def test_c_exact_knn_and_medoid_match_reference():
    f = golden("misc")
    x, q = gaussian(3000, 32, 0), gaussian(200, 32, 1)
    ids, ds = cref.exact_knn(x, q, 20, block=64)
    np.testing.assert_array_equal(ids, f["gt_ids"])
    np.testing.assert_array_equal(ds.astype(np.float32), f["gt_dists"])
    assert cref.medoid(x) == int(f["medoid32"])
    assert cref.medoid(lowrank(4000, 128, 12, 0.05, 7)) == int(f["medoid128"])


@pytest.mark.parametrize("seed,n,d,R,L,alpha,mb", [
    (1, 1500, 24, 12, 24, 1.2, 300),
    (2, 2000, 48, 20, 40, 1.0, 500),
    (3, 900, 17, 6, 10, 1.5, 100),
])
def test_c_build_matches_numpy_oracle_random(seed, n, d, R, L, alpha, mb):
    x = lowrank(n, d, 6, 0.1, seed)
    a = cref.build(x, R, L, alpha, max_batch=mb, threads=3)
    b = vamana.build(x, R, L, alpha, max_batch=mb)
    np.testing.assert_array_equal(a.adj, b.adj)
    assert a.entry == b.entry


def test_c_rabitq_search_matches_numpy_oracle_multibit():
    x, q = lowrank(2500, 40, 8, 0.1, 4), lowrank(60, 40, 8, 0.1, 5)
    g = vamana.build(x, 16, 32, 1.2)
    for bits in (2, 8):
        c, codes, meta = rabitq.fit(x, bits, 9)
        keys, hops, evals = cref.search_rabitq(g.adj, g.active, g.entry, cref.Quantized(c, codes, meta, bits, 9),
                                               q, 48)
        src = rabitq.QuantSource(codes, meta, bits, 40, *rabitq.bind(q, c, bits, 9))
        ref = search.beam_search(g.adj, g.active, g.entry, src, len(q), 48)
        for r, o in zip(cref.results(keys, hops, evals), ref):
            np.testing.assert_array_equal(r.frontier_ids, o.frontier_ids)
            np.testing.assert_array_equal(r.frontier_dists, o.frontier_dists)
            assert (r.hops, r.evals) == (o.hops, o.evals)


def test_c_search_validation_matches_reference_errors():
    x = gaussian(50, 8, 0)
    rows = cref.Rows(x)
    g = vamana.build(x, 4, 8, 1.2)
    with pytest.raises(ValueError, match="beam_width"):
        cref.search_exact(g.adj, g.active, g.entry, rows, x[:2], 0)
    with pytest.raises(ValueError, match="start vertex"):
        cref.search_exact(g.adj, g.active, g.entry, rows, x[:2], 4, starts=[0, 50])
    with pytest.raises(ValueError, match="empty graph"):
        cref.search_exact(g.adj, 0, 0, rows, x[:2], 4)


def test_c_recall_ground_truth_consistent_with_numpy():
    x, q = lowrank(5000, 32, 8, 0.05, 3), lowrank(100, 32, 8, 0.05, 4)
    i1, d1 = cref.exact_knn(x, q, 50, block=32)
    i2, d2 = knn.exact_knn(x, q, 50)
    np.testing.assert_array_equal(i1, i2)
    np.testing.assert_array_equal(d1.astype(np.float32), d2)
