"""Tensor-core donor screen (csrc/donor_tc.cu): the connectivity repair's donor
lists, and therefore the graphs, are identical with the screen (tcgen05 tf32 +
exact A1 re-rank) and with the exact CUDA-core scan (JB_DONOR_TC=0), and both
match the oracle restatement of the reference (build.py:185-224)."""

import os

import numpy as np
import pytest

from conftest import gaussian, lowrank
from oracle import vamana

pytestmark = pytest.mark.gpu

jb = pytest.importorskip("paper_2601_07048_b200")
import importlib  # noqa: E402

jbuild = importlib.import_module("paper_2601_07048_b200.build")


def _build(x, env, **kw):
    old = os.environ.get("JB_DONOR_TC")
    os.environ["JB_DONOR_TC"] = env
    try:
        jbuild.WORK[:] = 0
        g = jb.build(jb.VectorDataset(x), jb.BuildParams(**kw))
        return g, dict(zip(jbuild.WORK_FIELDS, (int(v) for v in jbuild.WORK)))
    finally:
        if old is None:
            del os.environ["JB_DONOR_TC"]
        else:
            os.environ["JB_DONOR_TC"] = old


# iid Gaussian rows bridge often (~25% of a batch at R=24); D = 100 leaves a
# partial last K chunk (TMA zero fill), D = 128 fills four, D = 36 one partial
@pytest.mark.parametrize("n,D,R", [(12000, 64, 24), (9000, 100, 16), (6000, 128, 32), (5000, 36, 12)])
def test_tensor_core_donors_identical_to_exact_scan(n, D, R):
    x = gaussian(n, D, 300 + D)
    kw = dict(degree_cap=R, build_beam_width=2 * R, alpha=1.2, max_batch=max(400, n // 4))
    gt, wt = _build(x, "1", **kw)
    ge, we = _build(x, "0", **kw)
    assert wt["bridges"] > 0 and wt["bridges"] == we["bridges"]
    assert wt["donor_tc_rows"] > 0, "the tensor-core screen did not run"
    assert we["donor_tc_rows"] == 0
    # the screen certifies almost every row (the rest are rescanned exactly)
    assert wt["donor_tc_redo"] <= 0.05 * wt["donor_tc_rows"], wt
    assert gt.entry_point == ge.entry_point
    np.testing.assert_array_equal(gt.degrees, ge.degrees)
    np.testing.assert_array_equal(gt.adjacency, ge.adjacency)


def test_tensor_core_donors_identical_to_oracle():
    x = lowrank(3000, 96, 6, 0.3, 311)
    og = vamana.build(x, R=12, L=24, alpha=1.2, max_batch=600)
    g, w = _build(x, "1", degree_cap=12, build_beam_width=24, alpha=1.2, max_batch=600)
    assert w["donor_tc_rows"] > 0
    assert g.entry_point == og.entry
    np.testing.assert_array_equal(g.degrees[:3000], og.deg)
    np.testing.assert_array_equal(g.adjacency[:3000], og.adj)
