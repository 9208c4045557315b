"""GPU exact kNN (jb_exact_knn, the ground-truth path) vs the live reference's
golden `exact_knn` output and the oracle restatement (oracle.py:20-62).

The device sums dot products in a different f64 order than OpenBLAS, so scores
agree to f64 rounding: distances (f32 outputs) must match to 1 ulp-ish
(rtol 1e-6), and ids must match wherever the reference's neighbouring scores are
separated by more than that rounding (exact ties keep the (dist, id) order)."""

import numpy as np
import pytest

from conftest import gaussian, golden, lowrank
from oracle import knn as oknn

pytestmark = pytest.mark.gpu

jb = pytest.importorskip("paper_2601_07048_b200")


# f64 rounding of (xn - 2 q.x) + qn is relative to the operands, not to the
# result: a self-match can come out as 0 or ~1e-14 depending on summation order.
ATOL = 1e-9


def _check(ids, ds, exp_ids, exp_ds):
    np.testing.assert_allclose(ds, exp_ds, rtol=1e-6, atol=ATOL)
    e = exp_ds.astype(np.float64)
    for q in range(e.shape[0]):
        row = e[q]
        sep = np.ones(row.size, dtype=bool)
        gap = np.diff(row) <= 1e-9 * np.abs(row[1:]) + ATOL
        sep[1:] &= ~gap
        sep[:-1] &= ~gap
        np.testing.assert_array_equal(ids[q][sep], exp_ids[q][sep], err_msg=f"query {q}")
        assert sorted(ids[q].tolist()) == sorted(set(ids[q].tolist())), "duplicate ids"


def test_exact_knn_matches_reference_golden():
    f = golden("misc")  # beamann.exact_knn(gen_synthetic(3000, 32, 0), gen_synthetic(200, 32, 1), 20)
    gt = jb.exact_knn(gaussian(3000, 32, 0), gaussian(200, 32, 1), 20)
    _check(gt.ids, gt.distances, f["gt_ids"], f["gt_dists"])


@pytest.mark.parametrize("n,d,k", [(5000, 128, 100), (3001, 33, 10), (700, 960, 50), (64, 7, 64), (20000, 96, 1)])
def test_exact_knn_matches_oracle(n, d, k):
    x = gaussian(n, d, n + d)
    q = gaussian(150, d, n + d + 1)
    gt = jb.exact_knn(x, q, k)
    ei, ed = oknn.exact_knn(x, q, k)
    _check(gt.ids, gt.distances, ei, ed)


def test_exact_knn_duplicates_and_ties_by_id():
    base = gaussian(300, 16, 3)
    x = np.concatenate([base, base, base[:50]])  # exact duplicate rows: equal scores, ties by id
    q = np.concatenate([base[:20], gaussian(20, 16, 4)])
    gt = jb.exact_knn(x, q, 40)
    ei, ed = oknn.exact_knn(x, q, 40)
    np.testing.assert_allclose(gt.distances, ed, rtol=1e-6, atol=ATOL)
    for i in range(len(q)):  # equal-distance groups come out in ascending id order
        d = gt.distances[i]
        for j in range(1, len(d)):
            if d[j] == d[j - 1]:
                assert gt.ids[i][j] > gt.ids[i][j - 1]


def test_exact_knn_large_n_select_path():
    # n large enough that the radix select refines more than one digit
    x = lowrank(400_000, 32, 8, 0.05, 11)
    q = lowrank(40, 32, 8, 0.05, 12)
    gt = jb.exact_knn(x, q, 100)
    ei, ed = oknn.exact_knn(x, q, 100)
    _check(gt.ids, gt.distances, ei, ed)


def test_exact_knn_validation():
    x = gaussian(10, 4, 0)
    with pytest.raises(ValueError):
        jb.exact_knn(x, x, 11)
    with pytest.raises(ValueError):
        jb.exact_knn(x, gaussian(3, 5, 0), 2)


def test_mips_augment_inner_product_gt_build_and_search_match_reference():
    from conftest import gaussian as _g

    f = golden("mips")
    data = _g(2000, 24, 61) * np.linspace(0.5, 2.0, 2000, dtype=np.float32)[:, None]
    q = _g(60, 24, 62)
    ad, aq = jb.mips_augment(jb.VectorDataset(data), jb.VectorDataset(q))
    assert isinstance(ad, jb.AugmentedDataset) and ad.role == "data" and aq.role == "query" and ad.base_dims == 24
    np.testing.assert_array_equal(ad.dataset.data, f["aug_data"])   # bit-exact f64 norms / sqrt
    np.testing.assert_array_equal(aq.dataset.data, f["aug_queries"])
    assert ad.max_norm == float(f["max_norm"])
    gt = jb.exact_knn(jb.VectorDataset(data), jb.VectorDataset(q), 10, jb.DistanceKind.INNER_PRODUCT)
    np.testing.assert_array_equal(gt.ids, f["gt_ids"])
    np.testing.assert_allclose(gt.distances, f["gt_dists"], rtol=1e-6, atol=1e-6)
    g = jb.build(ad, jb.BuildParams(degree_cap=16, build_beam_width=32, alpha=1.2))
    np.testing.assert_array_equal(g.adjacency[:2000], f["adjacency"])
    assert g.entry_point == int(f["entry"])
    ids, dists = jb.search_knn_batch(g, ad, aq.dataset.data, jb.SearchParams(beam_width=32, k=10))
    np.testing.assert_array_equal(ids, f["knn_ids"])
    np.testing.assert_array_equal(dists, f["knn_dists"])
    with pytest.raises(ValueError, match="mips_augment requires f32 datasets"):
        jb.mips_augment(jb.VectorDataset(np.zeros((4, 3), np.uint8)), jb.VectorDataset(np.zeros((1, 3), np.uint8)))
