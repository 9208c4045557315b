"""SPEC.md RaBitQ known answers and properties,
on the device fit/estimator. Host-only parts run on CPU."""

import numpy as np
import pytest

from conftest import gaussian, lowrank

jb = pytest.importorskip("paper_2601_07048_b200")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.parametrize("bits", [1, 2, 4, 8])
def test_pack_unpack_round_trip_and_storage(bits):
    rng = np.random.default_rng(bits)
    for d in (1, 7, 33, 128, 960):
        u = rng.integers(0, 2 ** bits, size=(5, d), dtype=np.uint8)
        packed = jb.rabitq.pack_codes(u, bits)
        assert packed.shape == (5, (d * bits + 7) // 8)
        np.testing.assert_array_equal(jb.rabitq.unpack_codes(packed, bits, d), u)
    # storage per vector: code bytes + (data_add, data_rescale) f32
    idx = jb.RaBitQIndex(128, 4, 0, np.zeros(128, np.float32), np.zeros((3, 64), np.uint8), np.zeros((3, 2), np.float32))
    assert idx.per_vector_bytes == 64 + 8
    idx960 = jb.RaBitQIndex(960, 4, 0, np.zeros(960, np.float32), np.zeros((2, 480), np.uint8),
                            np.zeros((2, 2), np.float32))
    assert idx960.per_vector_bytes == 488


def _estimates(idx, q):
    """Host restatement of the estimator (rabitq.py:235-244) from the device bind."""
    b = idx.bind(q[None, :])
    rot, qa, qs = b.rotated, b.query_add, b.query_sumq
    u = jb.rabitq.unpack_codes(idx.codes, idx.bits, idx.dims).astype(np.float32)
    dd = u @ rot[0]
    return qa[0] + idx.meta[:, 0] + idx.meta[:, 1] * (dd - qs[0])


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [1, 4, 8])
def test_zero_residual_row_has_zero_metadata(bits):
    a = gaussian(10, 32, 3)
    x = np.concatenate([a, -a, np.zeros((1, 32), np.float32)])  # mean 0: the last row is the centroid
    idx = jb.rabitq_fit(jb.VectorDataset(x), bits=bits, seed=2)
    np.testing.assert_array_equal(idx.centroid, np.zeros(32, np.float32))
    np.testing.assert_array_equal(idx.meta[-1], [0.0, 0.0])
    mid = 1 << (bits - 1)
    np.testing.assert_array_equal(jb.rabitq.unpack_codes(idx.codes[-1:], bits, 32)[0], np.full(32, mid))


@pytest.mark.gpu
@pytest.mark.parametrize("bits,min_rho", [(8, 0.99), (4, 0.99), (1, 0.8)])
def test_estimator_rank_correlation(bits, min_rho):
    from scipy.stats import spearmanr

    x = gaussian(4000, 128, 11)
    q = gaussian(3, 128, 12)
    idx = jb.rabitq_fit(jb.VectorDataset(x), bits=bits, seed=5)
    for qq in q:
        est = _estimates(idx, qq)
        exact = ((x.astype(np.float64) - qq) ** 2).sum(axis=1)
        rho = spearmanr(est, exact).correlation
        assert rho >= min_rho, (bits, rho)
        rel = (est - exact) / exact
        assert abs(float(np.mean(rel))) < 0.05  # unbiased on average


@pytest.mark.gpu
def test_960d_m4_rerank_recall_within_3_points_of_exact():
    """SPEC.md:625 at reduced N: 960-d, m = 4 (488 B per vector) + fp32 rerank."""
    x = lowrank(5000, 960, 24, 0.05, 21)
    q = lowrank(200, 960, 24, 0.05, 22)
    ds = jb.VectorDataset(x)
    g = jb.build(ds, jb.BuildParams(degree_cap=24, build_beam_width=48, alpha=1.2))
    idx = jb.rabitq_fit(ds, bits=4, seed=3)
    assert idx.per_vector_bytes == 488
    gt = jb.exact_knn(ds, jb.VectorDataset(q), 10)
    ex, _ = jb.search_knn_batch(g, ds, q, jb.SearchParams(beam_width=48, k=10))
    rq, _ = jb.search_knn_batch(g, idx, q, jb.SearchParams(beam_width=48, k=10, rerank=True), exact_data=ds)
    r_exact, r_quant = jb.recall_at_k(ex, gt, 10), jb.recall_at_k(rq, gt, 10)
    assert r_quant >= r_exact - 0.03, (r_exact, r_quant)


@pytest.mark.gpu
def test_column_mean_bit_exact_on_ragged_shapes():
    """jb_column_mean_f32 = x.astype(f64).mean(axis=0).astype(f32) (rabitq.py:273) bit for bit:
    row counts off the 512-row smem tile and column counts off the 8-column group."""
    import torch

    from paper_2601_07048_b200 import _lib

    rng = np.random.default_rng(11)
    for n, d in ((1, 3), (5, 8), (511, 33), (70001, 33), (3000, 960), (100003, 128)):
        x = (rng.standard_normal((n, d)) * rng.uniform(0.1, 100.0, size=d)).astype(np.float32)
        want = x.astype(np.float64).mean(axis=0).astype(np.float32)
        xd = torch.from_numpy(x).cuda()
        out = torch.empty(d, dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().jb_column_mean_f32(_lib.ptr(xd), n, d, _lib.ptr(out), _lib.stream_ptr()))
        got = out.cpu().numpy()
        assert got.tobytes() == want.tobytes(), (n, d)


@pytest.mark.gpu
def test_row_sq_norms_matches_reference_einsum():
    """core.py:161-166: einsum('nd,nd->n') bit for bit on f32 rows, integer-exact int64 on u8."""
    rng = np.random.default_rng(5)
    for d in (1, 7, 33, 128, 960):
        x = (rng.standard_normal((300, d)) * 3).astype(np.float32)
        got = jb.row_sq_norms(x)
        assert got.dtype == np.float32
        assert got.tobytes() == np.einsum("nd,nd->n", x, x).tobytes()
        u = rng.integers(0, 256, size=(200, d), dtype=np.uint8)
        w = u.astype(np.int64)
        gu = jb.row_sq_norms(u)
        assert gu.dtype == np.int64 and np.array_equal(gu, np.einsum("nd,nd->n", w, w))
    with pytest.raises(ValueError):
        jb.row_sq_norms(np.zeros((3, 4), np.float64))
