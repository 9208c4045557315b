"""Int8 screen of the exact search (extension, jb_search_args.screen): a new
neighbour proven worse than the full beam's worst key is dropped without its f32
row. Frontier, trace and evals must equal the unscreened search, and graphs
built with the screen equal the oracle's and the unscreened build's. The staged
(non-L2-resident) exact path is forced with JB_EXACT_DIRECT=0."""

import os

import numpy as np
import pytest

from conftest import gaussian, lowrank
from oracle import cref

pytestmark = pytest.mark.gpu

jb = pytest.importorskip("paper_2601_07048_b200")


class _env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update(self.kv)

    def __exit__(self, *exc):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_screen_records_bound_the_quantisation_error():
    import torch

    from paper_2601_07048_b200 import _lib

    for n, d in ((1000, 128), (300, 33), (50, 960)):
        x = lowrank(n, d, 12, 0.05, 3)
        ds = jb.VectorDataset(x)
        rec, cen = ds.device_screen()
        rb = int(_lib.lib().jb_screen_record_bytes(d))
        assert rec.shape == (n, rb) and rb == ((d + 15) // 16) * 16 + 16
        r = rec.cpu().numpy()
        c = cen.cpu().numpy().astype(np.float64)
        b = r[:, :d].view(np.int8).astype(np.float64)
        meta = r[:, rb - 16:].copy().view(np.float32)
        s, bb, eps, nx = meta[:, 0].astype(np.float64), meta[:, 1], meta[:, 2].astype(np.float64), meta[:, 3]
        err = np.sqrt(((s[:, None] * b - (x.astype(np.float64) - c)) ** 2).sum(1))
        assert (err <= eps).all()
        assert np.array_equal(bb, (b ** 2).sum(1).astype(np.float32))
        assert (r[:, d:rb - 16] == 0).all()
        assert np.array_equal(nx, ds.device().norms.cpu().numpy())
        assert np.abs(b).max() <= 127


@pytest.mark.parametrize("L", [16, 64, 200])
def test_screened_search_identical(L):
    x = lowrank(30000, 128, 16, 0.05, 5)
    q = lowrank(300, 128, 16, 0.05, 6)
    ds = jb.VectorDataset(x)
    g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=48, alpha=1.2))
    from paper_2601_07048_b200 import search as js

    outs = []
    for scr in ("0", "1"):
        with _env(JB_EXACT_DIRECT="0", JB_SEARCH_SCREEN=scr):
            outs.append(js.run_beam_searches(g, ds, q, L))
    for a, b in zip(*outs):
        assert np.array_equal(a.frontier_ids, b.frontier_ids)
        assert np.array_equal(a.frontier_dists, b.frontier_dists)
        assert np.array_equal(a.visited_ids, b.visited_ids)
        assert a.stats == b.stats


@pytest.mark.parametrize("D,seed", [(128, 1), (96, 2), (40, 3)])
def test_screened_build_identical_to_oracle_and_unscreened(D, seed):
    x = lowrank(6000, D, 12, 0.05, seed) if D != 40 else gaussian(6000, D, seed)
    p = jb.BuildParams(degree_cap=24, build_beam_width=40, alpha=1.2, max_batch=2000)
    graphs = []
    for scr in ("0", "1"):
        with _env(JB_EXACT_DIRECT="0", JB_SCREEN=scr):
            graphs.append(jb.build(jb.VectorDataset(x), p))
    ref = cref.build(x, 24, 40, 1.2, max_batch=2000)
    for g in graphs:
        n = g.active_count
        assert np.array_equal(g.host_adjacency()[:n], ref.adj[:n])
        assert np.array_equal(g.degrees[:n], ref.deg[:n])
        assert g.entry_point == ref.entry


@pytest.mark.parametrize("D,R", [(33, 16), (50, 24), (200, 24), (300, 16), (96, 64)])
def test_screened_search_identical_shapes(D, R):
    """Unaligned rows (D % 4 != 0), rows staged in several 128-element chunks with a
    partial 16-block tail (D = 200, 300: the split A1 chains cross chunk boundaries),
    and R = 64 (two neighbour chunks per hop, the worst key re-read between them)."""
    x = lowrank(8000, D, 12, 0.05, D + R)
    q = lowrank(120, D, 12, 0.05, D + R + 1)
    ds = jb.VectorDataset(x)
    g = jb.build(ds, jb.BuildParams(degree_cap=R, build_beam_width=40, alpha=1.2, max_batch=2000))
    from paper_2601_07048_b200 import search as js

    outs = []
    for scr in ("0", "1"):
        with _env(JB_EXACT_DIRECT="0", JB_SEARCH_SCREEN=scr, JB_SCREEN_FORCE="1"):
            outs.append(js.run_beam_searches(g, ds, q, 48))
    for a, b in zip(*outs):
        assert np.array_equal(a.frontier_ids, b.frontier_ids)
        assert np.array_equal(a.frontier_dists, b.frontier_dists)
        assert np.array_equal(a.visited_ids, b.visited_ids)
        assert a.stats == b.stats


@pytest.mark.parametrize("D", [200, 33])
def test_screened_build_chunked_and_unaligned_rows_identical_to_oracle(D):
    x = lowrank(3000, D, 12, 0.05, 7 * D)
    p = jb.BuildParams(degree_cap=16, build_beam_width=32, alpha=1.2, max_batch=1000)
    with _env(JB_EXACT_DIRECT="0", JB_SCREEN_FORCE="1"):
        g = jb.build(jb.VectorDataset(x), p)
    ref = cref.build(x, 16, 32, 1.2, max_batch=1000)
    n = g.active_count
    assert np.array_equal(g.host_adjacency()[:n], ref.adj[:n])
    assert g.entry_point == ref.entry


@pytest.mark.parametrize("D", [96, 128])
def test_screen_next_hop_staging_identical(D):
    """snext mode (the speculative next hop's records staged in smem one hop ahead,
    the default beyond 3 x L2 of records) forced on small data: identical searches
    and builds."""
    x = lowrank(8000, D, 12, 0.05, 3 * D)
    q = lowrank(150, D, 12, 0.05, 3 * D + 1)
    ds = jb.VectorDataset(x)
    p = jb.BuildParams(degree_cap=24, build_beam_width=40, alpha=1.2, max_batch=2000)
    from paper_2601_07048_b200 import search as js

    with _env(JB_EXACT_DIRECT="0", JB_SCREEN_NEXT="0"):
        g0 = jb.build(ds, p)
        r0 = js.run_beam_searches(g0, ds, q, 64)
    with _env(JB_EXACT_DIRECT="0", JB_SCREEN_NEXT="1"):
        g1 = jb.build(ds, p)
        r1 = js.run_beam_searches(g0, ds, q, 64)
    n = g0.active_count
    assert np.array_equal(g0.host_adjacency()[:n], g1.host_adjacency()[:n])
    for a, b in zip(r0, r1):
        assert np.array_equal(a.frontier_ids, b.frontier_ids)
        assert np.array_equal(a.visited_ids, b.visited_ids)
        assert a.stats == b.stats
