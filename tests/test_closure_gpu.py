"""Prune closure (extension, jb_insert_args.closure): a row written by a robust
prune at alpha^2 has no member pruning a later one, so the owner merge of such a
row only tests the pairs involving its fresh sources. Graphs must be identical
with the closure on and off (JB_CLOSURE=0), and a row written outside the
library's prune kernels (host edits, appends, bridges) must not be trusted."""

import importlib
import os

import numpy as np
import pytest

from conftest import gaussian, lowrank
from oracle import cref

pytestmark = pytest.mark.gpu

jb = pytest.importorskip("paper_2601_07048_b200")
jbuild = importlib.import_module("paper_2601_07048_b200.build")


def _stream(x, env, params, n0, steps):
    old = os.environ.get("JB_CLOSURE")
    os.environ["JB_CLOSURE"] = env
    try:
        ds = jb.VectorDataset(x)
        g = jb.GraphIndex(len(x), params.degree_cap)
        jb.insert_stream(g, ds, range(0, n0), params)
        pos = n0
        for s in steps:
            jb.insert_stream(g, ds, range(pos, pos + s), params)
            pos += s
        return g
    finally:
        if old is None:
            del os.environ["JB_CLOSURE"]
        else:
            os.environ["JB_CLOSURE"] = old


@pytest.mark.parametrize("D,kind", [(64, "lowrank"), (128, "gaussian"), (96, "lowrank")])
def test_closure_graphs_identical(D, kind):
    x = lowrank(24000, D, 12, 0.05, 400 + D) if kind == "lowrank" else gaussian(24000, D, 400 + D)
    p = jb.BuildParams(degree_cap=24, build_beam_width=48, alpha=1.2, max_batch=2000)
    on = _stream(x, "1", p, 8000, [4000, 6000, 6000])
    off = _stream(x, "0", p, 8000, [4000, 6000, 6000])
    assert on.entry_point == off.entry_point
    np.testing.assert_array_equal(on.degrees, off.degrees)
    np.testing.assert_array_equal(on.adjacency, off.adjacency)


def test_host_edits_invalidate_closure():
    """A host-side row edit between inserts must reset the closure: the graph then
    matches the oracle given the same edit."""
    x = lowrank(6000, 64, 8, 0.05, 41)
    p = jb.BuildParams(degree_cap=16, build_beam_width=32, alpha=1.2, max_batch=1000)
    ds = jb.VectorDataset(x)
    g = jb.GraphIndex(6000, 16)
    jb.insert_stream(g, ds, range(0, 3000), p)
    og = cref.Graph(6000, 16)
    og.adj[:] = g.adjacency
    og.deg[:] = g.degrees
    og.active, og.entry = g.active_count, g.entry_point
    # replace some full rows on the host with random (valid, not prune-closed) sets:
    # a stale closure flag would skip their existing-existing pair tests
    rng = np.random.default_rng(7)
    for u in range(0, 3000, 7):
        d = int(g.degrees[u])
        pool = np.setdiff1d(np.arange(3000), [u])
        row = rng.choice(pool, size=d, replace=False).astype(np.int32)
        g.set_neighbors(u, row.tolist())
        og.adj[u, :] = -1
        og.adj[u, :d] = row
    jb.insert_stream(g, ds, range(3000, 6000), p)
    cref.insert_stream(og, cref.Rows(x), 3000, 6000, 32, 1.2, 1000)
    assert g.entry_point == og.entry
    np.testing.assert_array_equal(g.degrees, og.deg)
    np.testing.assert_array_equal(g.adjacency, og.adj)


def test_other_dataset_resets_closure():
    """The closure is tied to the dataset it was computed against."""
    x = lowrank(4000, 64, 8, 0.05, 43)
    p = jb.BuildParams(degree_cap=16, build_beam_width=32, alpha=1.2, max_batch=1000)
    g = jb.GraphIndex(4000, 16)
    ds1 = jb.VectorDataset(x)
    jb.insert_stream(g, ds1, range(0, 2000), p)
    tok1 = g._closure_key
    jb.insert_stream(g, jb.VectorDataset(x.copy()), range(2000, 4000), p)
    assert g._closure_key != tok1


def test_closure_global_row_path_identical():
    """beamann's default R = 64 at D = 128: candidate sets too large to stage, the
    owner merge prunes from global rows (prune_closed_global for closed rows)."""
    x = lowrank(16000, 128, 12, 0.05, 47)
    p = jb.BuildParams(degree_cap=64, build_beam_width=128, alpha=1.2, max_batch=2000)
    on = _stream(x, "1", p, 6000, [4000, 6000])
    off = _stream(x, "0", p, 6000, [4000, 6000])
    assert on.entry_point == off.entry_point
    np.testing.assert_array_equal(on.degrees, off.degrees)
    np.testing.assert_array_equal(on.adjacency, off.adjacency)
